set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tp_fused.py -q -x -k "layer or fused_grad or operators" > gpurun_out/pytest_ef.log 2>&1
echo "exit $?" >> gpurun_out/pytest_ef.log
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_ef0.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ef0_$i.json 2>/dev/null
HXM_LIB=$PWD/ab/libhexamoe_ef1.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ef1_$i.json 2>/dev/null
done
