set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "operators_at_scale" > gpurun_out/pytest_op.log 2>&1
echo "exit $?" >> gpurun_out/pytest_op.log
