# Full default bench + reference arm + other configs + ncu evidence (one GPU).
set -x
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
python bench.py --config c3 --no-cpu-baseline --steps 30 > gpurun_out/bench_c3.json 2>&1
python bench.py --config c4 --no-cpu-baseline --steps 10 > gpurun_out/bench_c4.json 2>&1
python bench.py --config c5 --no-cpu-baseline --steps 30 > gpurun_out/bench_c5.json 2>&1
python bench.py --config c5 --no-cpu-baseline --steps 30 --capacity-factor 1.25 > gpurun_out/bench_c5_cf125.json 2>&1
python bench.py --config c1 --no-cpu-baseline --steps 30 > gpurun_out/bench_c1.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --no-graph --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"umma_kernel|prologue|colsum" -s 9 -c 9 -o gpurun_out/prof_full python bench.py --no-graph --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
