set -x
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --mode data_centric --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dc1.json 2> gpurun_out/bench_dc1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --mode model_centric --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mc1.json 2> gpurun_out/bench_mc1.err
timeout 300 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err; echo "gpus2 exit $?" >> gpurun_out/bench_g2.err
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_nccl_capi.py tests/test_gpu_tp_fused.py tests/test_gpu_shards.py -q > gpurun_out/pytest_dist.log 2>&1; echo "exit $?" >> gpurun_out/pytest_dist.log
