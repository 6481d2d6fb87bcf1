set -x
HXM_WIDE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"umma_wide" -s 0 -c 2 -o gpurun_out/prof_wide python bench.py --no-graph --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_wide.log 2>&1
HXM_WIDE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"umma_kernel<192, 0" -s 0 -c 2 -o gpurun_out/prof_n192 python bench.py --no-graph --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_n192.log 2>&1
