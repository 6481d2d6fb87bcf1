set -x
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -q -k "skew" > gpurun_out/pytest_skew.log 2>&1
echo "exit $?" >> gpurun_out/pytest_skew.log
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/tma_bw.cu -lcuda -o /tmp/tma_bw && timeout 300 /tmp/tma_bw > gpurun_out/tma_bw.log 2>&1
