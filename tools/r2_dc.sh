set -x
timeout 900 python -m pytest tests/test_gpu_shards.py tests/test_gpu_dist.py tests/test_gpu_tp_fused.py -q -rf > gpurun_out/pytest_dc.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_dc.log
timeout 600 python bench.py --mode data_centric --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3_dc1.json 2> gpurun_out/bench_c3_dc1.err
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
