set -x
timeout 900 ncu --set full --clock-control none -k regex:"umma|prologue|colsum" -s 9 -c 9 -o gpurun_out/prof_c3 python bench.py --config c3 --no-graph --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --no-graph --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3_final.json 2>/dev/null
