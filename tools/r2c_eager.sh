set -x
timeout 300 python bench.py --no-graph --no-cpu-baseline --steps 30 > gpurun_out/bench_eager.json 2> gpurun_out/bench_eager.err
