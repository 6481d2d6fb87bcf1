set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_shards.py tests/test_gpu_tp_fused.py -q -rf -x > gpurun_out/pytest_sk.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_sk.log
for i in 1 2; do
HXM_STREAMK=0 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_sk0_$i.json 2>/dev/null
HXM_STREAMK=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_sk1_$i.json 2>/dev/null
done
HXM_STREAMK=0 timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3_sk0.json 2>/dev/null
HXM_STREAMK=1 timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3_sk1.json 2>/dev/null
