set -x
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 30 > gpurun_out/bench_c1_final.json 2>/dev/null
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3_final.json 2>/dev/null
timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 10 > gpurun_out/bench_c4_final.json 2>/dev/null
timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 20 > gpurun_out/bench_c5_final.json 2>/dev/null
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --mode data_centric --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dc1_final.json 2>/dev/null
