set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_tp_fused.py tests/test_gpu_shards.py -q -x > gpurun_out/pytest_gz.log 2>&1
echo "exit $?" >> gpurun_out/pytest_gz.log
for i in 1 2 3; do
HXM_GW2_ZERO=0 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_gz0_$i.json 2>gpurun_out/bench_gz0_$i.err
HXM_GW2_ZERO=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_gz1_$i.json 2>gpurun_out/bench_gz1_$i.err
done
