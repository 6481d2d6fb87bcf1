# iteration: gpu tests + c2 bench (+ extra args passed as $@ to pytest -k)
set -x
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 1800 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
HXM_PRO1=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_pro3.json 2> gpurun_out/bench_c2_pro3.err
timeout 300 python tools/prologue_ts.py > gpurun_out/prologue_ts.txt 2>&1
