set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "layer or ess or gb2" > gpurun_out/pytest_pro.log 2>&1
echo "exit $?" >> gpurun_out/pytest_pro.log
HXM_LIB=$PWD/ab/libhexamoe_old.so true
for i in 1 2 3; do
timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_pro_$i.json 2>gpurun_out/bench_pro_$i.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_pro.csv python bench.py --no-graph --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
