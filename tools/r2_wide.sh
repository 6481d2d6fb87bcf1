set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "layer or c2" > gpurun_out/pytest_wide.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_wide.log
for i in 1 2; do
HXM_WIDE=0 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_w0_$i.json 2>/dev/null
HXM_WIDE=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_w1_$i.json 2>gpurun_out/bench_w1_$i.err
done
