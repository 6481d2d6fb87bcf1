set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_chain.py tests/test_gpu_tp_fused.py tests/test_gpu_shards.py -q -x > gpurun_out/pytest_z.log 2>&1
echo "exit $?" >> gpurun_out/pytest_z.log
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_pw1.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_z0_$i.json 2>gpurun_out/bench_z0_$i.err
HXM_LIB=$PWD/ab/libhexamoe_z1.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_z1_$i.json 2>gpurun_out/bench_z1_$i.err
done
