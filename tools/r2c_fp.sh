set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q -x -k "layer or c2 or skew or edge" > gpurun_out/pytest_fp.log 2>&1
echo "exit $?" >> gpurun_out/pytest_fp.log
HXM_LIB=$PWD/ab/libhexamoe_fp0.so timeout 600 python tools/chain_check.py save off > gpurun_out/fp_off.log 2>&1
HXM_LIB=$PWD/ab/libhexamoe_fp1.so timeout 600 python tools/chain_check.py save on > gpurun_out/fp_on.log 2>&1
python tools/chain_check.py compare off on > gpurun_out/fp_cmp.log 2>&1
rm -f /tmp/chain_*.pt
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_fp0.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_fp0_$i.json 2>gpurun_out/bench_fp0_$i.err
HXM_LIB=$PWD/ab/libhexamoe_fp1.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_fp1_$i.json 2>gpurun_out/bench_fp1_$i.err
done
