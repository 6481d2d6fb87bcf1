set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "layer or c2" > gpurun_out/pytest_pw.log 2>&1
echo "exit $?" >> gpurun_out/pytest_pw.log
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_pw0.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_pw0_$i.json 2>gpurun_out/bench_pw0_$i.err
HXM_LIB=$PWD/ab/libhexamoe_pw1.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_pw1_$i.json 2>gpurun_out/bench_pw1_$i.err
done
HXM_LIB=$PWD/ab/libhexamoe_pw1.so timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_pw1_c3.json 2>/dev/null
