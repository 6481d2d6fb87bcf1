# chained fwd + bwd: bit-identity, layer parity, bench A/B, trace, launch list
set -x
HXM_CHAIN=0 HXM_CHAIN_BWD=0 timeout 600 python tools/chain_check.py save off > gpurun_out/chain_off.log 2>&1
HXM_CHAIN=1 HXM_CHAIN_BWD=1 timeout 600 python tools/chain_check.py save on > gpurun_out/chain_on.log 2>&1
python tools/chain_check.py compare off on > gpurun_out/chain_cmp.log 2>&1
rm -f /tmp/chain_*.pt
HXM_CHAIN_BWD=1 HXM_CHAIN_TRACE=1 timeout 300 python tools/chain_trace.py > gpurun_out/chain_trace.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q -x -k "layer or c2 or c4 or c5" > gpurun_out/pytest_chain.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_chain.log
for i in 1 2; do
HXM_CHAIN=0 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ch0_$i.json 2>gpurun_out/bench_ch0_$i.err
HXM_CHAIN=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ch1_$i.json 2>gpurun_out/bench_ch1_$i.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_chain.csv python bench.py --no-graph --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
