set -x
HXM_LIB=$PWD/ab/libhexamoe_x1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py -q -x -k "layer or c2 or operators or chain" > gpurun_out/pytest_wu2.log 2>&1
echo "exit $?" >> gpurun_out/pytest_wu2.log
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_x0.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_x0_$i.json 2>/dev/null
HXM_LIB=$PWD/ab/libhexamoe_x1.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_x1_$i.json 2>/dev/null
done
