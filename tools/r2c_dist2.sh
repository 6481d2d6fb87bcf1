set -x
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --mode data_centric --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dc1.json 2> gpurun_out/bench_dc1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --mode model_centric --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mc1.json 2> gpurun_out/bench_mc1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --mode data_centric --no-fused --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dc1nf.json 2> gpurun_out/bench_dc1nf.err
