set -x
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_base.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_nb0_$i.json 2>gpurun_out/bench_nb0_$i.err
HXM_LIB=$PWD/ab/libhexamoe_nb.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_nb1_$i.json 2>gpurun_out/bench_nb1_$i.err
done
