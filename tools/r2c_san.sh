set -x
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -q -rf --timeout 2000 > gpurun_out/pytest_san.log 2>&1
echo "exit $?" >> gpurun_out/pytest_san.log
