set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py -q -x -k "layer or c2 or chain" > gpurun_out/pytest_tr.log 2>&1
echo "exit $?" >> gpurun_out/pytest_tr.log
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_tr0.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_tr0_$i.json 2>gpurun_out/bench_tr0_$i.err
HXM_LIB=$PWD/ab/libhexamoe_tr1.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_tr1_$i.json 2>gpurun_out/bench_tr1_$i.err
done
for c in c1 c3 c5; do
HXM_LIB=$PWD/ab/libhexamoe_tr0.so timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/bench_tr0_$c.json 2>/dev/null
HXM_LIB=$PWD/ab/libhexamoe_tr1.so timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/bench_tr1_$c.json 2>/dev/null
done
