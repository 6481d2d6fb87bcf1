set -x
timeout 1500 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py tests/test_gpu_sanitizer.py -q > gpurun_out/pytest_fix.log 2>&1
echo "exit $?" >> gpurun_out/pytest_fix.log
HXM_CHAIN=1 HXM_CHAIN_BWD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q > gpurun_out/pytest_fix_chain.log 2>&1
echo "exit $?" >> gpurun_out/pytest_fix_chain.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_fix_$i.json 2>/dev/null; done
