# bench line, reference arm, launch list and ncu --set full of one c2 step (no tests)
set -x
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --no-graph --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"umma|prologue|colsum" -s 9 -c 9 -o gpurun_out/prof_full python bench.py --no-graph --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
