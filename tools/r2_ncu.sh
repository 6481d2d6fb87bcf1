set -x
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c2.csv python bench.py --no-graph --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prologue|colsum" -s 3 -c 3 -o gpurun_out/prof_pro python bench.py --no-graph --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
