set -x
HXM_CHAIN_BWD=1 HXM_CHAIN_TRACE=1 timeout 300 python tools/chain_trace.py > gpurun_out/chain_trace.log 2>&1
for i in 1 2; do
HXM_CHAIN=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ch1_$i.json 2>gpurun_out/bench_ch1_$i.err
HXM_CHAIN_BWD=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ch2_$i.json 2>gpurun_out/bench_ch2_$i.err
done
timeout 900 python -m pytest tests/test_gpu_chain.py -q -x > gpurun_out/pytest_chain.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_chain.log
