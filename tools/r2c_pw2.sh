set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_chain.py -q -x -k "layer or c2 or chain or skew" > gpurun_out/pytest_pw2.log 2>&1
echo "exit $?" >> gpurun_out/pytest_pw2.log
HXM_LIB=$PWD/ab/libhexamoe_pw0.so timeout 600 python tools/chain_check.py save off > gpurun_out/pw2_off.log 2>&1
HXM_LIB=$PWD/ab/libhexamoe_pw1.so timeout 600 python tools/chain_check.py save on > gpurun_out/pw2_on.log 2>&1
python tools/chain_check.py compare off on > gpurun_out/pw2_cmp.log 2>&1
rm -f /tmp/chain_*.pt
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_pw0.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_pwb0_$i.json 2>gpurun_out/bench_pwb0_$i.err
HXM_LIB=$PWD/ab/libhexamoe_pw1.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_pwb1_$i.json 2>gpurun_out/bench_pwb1_$i.err
done
