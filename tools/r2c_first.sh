# Round-2 (session 3) first GPU pass: tests, smoke, wide A/B bench, launch list.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 1500 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
for i in 1 2; do
HXM_WIDE=0 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_w0_$i.json 2>gpurun_out/bench_w0_$i.err
HXM_WIDE=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_w1_$i.json 2>gpurun_out/bench_w1_$i.err
done
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --no-graph --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
