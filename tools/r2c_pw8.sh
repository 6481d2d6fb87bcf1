set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q -x -k "bf16_vs_oracle or c3 or c4 or edge" > gpurun_out/pytest_pw8.log 2>&1
echo "exit $?" >> gpurun_out/pytest_pw8.log
HXM_EPI16=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bf16_vs_oracle or c2" >> gpurun_out/pytest_pw8.log 2>&1
echo "epi16=0 exit $?" >> gpurun_out/pytest_pw8.log
for i in 1 2; do
HXM_LIB=$PWD/ab/libhexamoe_base.so timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3b_$i.json 2>/dev/null
HXM_LIB=$PWD/ab/libhexamoe_pw8.so timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3n_$i.json 2>/dev/null
HXM_LIB=$PWD/ab/libhexamoe_pw8.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_c2n_$i.json 2>/dev/null
HXM_EPI16=0 HXM_LIB=$PWD/ab/libhexamoe_pw8.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_c2e8_$i.json 2>/dev/null
done
