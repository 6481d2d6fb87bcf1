set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32 or c1 or edge or chain_rule or layer" > gpurun_out/pytest_c1cs.log 2>&1
echo "exit $?" >> gpurun_out/pytest_c1cs.log
for i in 1 2 3; do
HXM_FUSE_GB1=0 timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 50 > gpurun_out/bench_cs0_$i.json 2>/dev/null
timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 50 > gpurun_out/bench_cs1_$i.json 2>/dev/null
done
