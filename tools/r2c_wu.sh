set -x
HXM_LIB=$PWD/ab/libhexamoe_w1.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "layer or c2 or operators" > gpurun_out/pytest_wu.log 2>&1
echo "exit $?" >> gpurun_out/pytest_wu.log
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_w0.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_w0_$i.json 2>/dev/null
HXM_LIB=$PWD/ab/libhexamoe_w1.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_w1_$i.json 2>/dev/null
done
