set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q -x -k "f32 or c1 or fp32 or esmm or estmm or esfk" > gpurun_out/pytest_c1.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_c1.log
for i in 1 2; do
HXM_SIMT_DENSE=0 timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 50 > gpurun_out/bench_c1d0_$i.json 2>gpurun_out/bench_c1d0_$i.err
timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 50 > gpurun_out/bench_c1d1_$i.json 2>gpurun_out/bench_c1d1_$i.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c1.csv python bench.py --config c1 --no-graph --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
