# ncu launch list of one bench step (cold-cache, serialised) -> gpurun_out/launches_$1.csv
cfg=${1:-c2}
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$cfg.csv python bench.py --config $cfg --no-graph --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_$cfg.csv
