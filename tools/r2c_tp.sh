set -x
timeout 900 python -m pytest tests/test_gpu_tp_fused.py tests/test_gpu_shards.py tests/test_gpu_dist.py -q > gpurun_out/pytest_tp.log 2>&1
echo "exit $?" >> gpurun_out/pytest_tp.log
