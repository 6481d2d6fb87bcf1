set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bf16_vs_oracle or edge" > gpurun_out/pytest_edge.log 2>&1
echo "exit $?" >> gpurun_out/pytest_edge.log
HXM_CHAIN=1 HXM_CHAIN_BWD=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bf16_vs_oracle or edge" >> gpurun_out/pytest_edge.log 2>&1
echo "chain exit $?" >> gpurun_out/pytest_edge.log
