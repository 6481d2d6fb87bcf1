# Other configs: bench lines + launch lists; c5 no-drop conventional; prologue ncu.
set -x
for c in c1 c3 c5; do
timeout 600 python bench.py --config $c --no-cpu-baseline --steps 30 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --no-graph --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 10 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 30 --capacity-factor 1.25 > gpurun_out/bench_c5_cf125.json 2> gpurun_out/bench_c5_cf125.err
timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 10 --capacity-factor 32 > gpurun_out/bench_c5_cf32.json 2> gpurun_out/bench_c5_cf32.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prologue|ess_kernel|simt" -s 0 -c 12 -o gpurun_out/prof_pro python bench.py --config c1 --no-graph --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_pro_c1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prologue" -s 2 -c 2 -o gpurun_out/prof_pro_c2 python bench.py --no-graph --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_pro_c2.log 2>&1
