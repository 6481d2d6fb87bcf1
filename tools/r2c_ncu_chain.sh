set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"umma_chain" -s 2 -c 2 -o gpurun_out/prof_chain python bench.py --no-graph --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_chain.log 2>&1
