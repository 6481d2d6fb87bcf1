set -x
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_b2.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_b2_$i.json 2>/dev/null
HXM_LIB=$PWD/ab/libhexamoe_b3.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_b3_$i.json 2>/dev/null
done
