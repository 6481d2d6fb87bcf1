set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_sanitizer.py -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/prologue_ts.py > gpurun_out/prologue_ts.txt 2>&1
HXM_PRO1=0 timeout 300 python tools/prologue_ts.py > gpurun_out/prologue_ts_old.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
