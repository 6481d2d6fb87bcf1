# chained fwd + bwd (F' by TMA through the chunk buffer): bit-identity, trace, bench A/B
set -x
HXM_CHAIN=0 HXM_CHAIN_BWD=0 timeout 600 python tools/chain_check.py save off > gpurun_out/chain_off.log 2>&1
HXM_CHAIN=1 HXM_CHAIN_BWD=1 timeout 600 python tools/chain_check.py save on > gpurun_out/chain_on.log 2>&1
python tools/chain_check.py compare off on > gpurun_out/chain_cmp.log 2>&1
rm -f /tmp/chain_*.pt
HXM_CHAIN_BWD=1 HXM_CHAIN_TRACE=1 timeout 300 python tools/chain_trace.py > gpurun_out/chain_trace.log 2>&1
for i in 1 2; do
HXM_CHAIN=0 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ch0_$i.json 2>gpurun_out/bench_ch0_$i.err
HXM_CHAIN=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ch1_$i.json 2>gpurun_out/bench_ch1_$i.err
HXM_CHAIN_BWD=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ch2_$i.json 2>gpurun_out/bench_ch2_$i.err
HXM_CHAIN_BWD=1 HXM_CHAIN_FPT=0 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_ch3_$i.json 2>gpurun_out/bench_ch3_$i.err
done
