set -x
HXM_WIDE_EST=0 timeout 600 python tools/chain_check.py save off > gpurun_out/west_off.log 2>&1
HXM_WIDE_EST=1 timeout 600 python tools/chain_check.py save on > gpurun_out/west_on.log 2>&1
python tools/chain_check.py compare off on > gpurun_out/west_cmp.log 2>&1
rm -f /tmp/chain_*.pt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q -x > gpurun_out/pytest_west.log 2>&1
echo "exit $?" >> gpurun_out/pytest_west.log
for i in 1 2 3; do
HXM_WIDE_EST=0 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_we0_$i.json 2>gpurun_out/bench_we0_$i.err
HXM_WIDE_EST=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_we1_$i.json 2>gpurun_out/bench_we1_$i.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_west.csv python bench.py --no-graph --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
