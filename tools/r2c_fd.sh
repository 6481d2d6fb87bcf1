set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q -x -k "layer or c2 or c5 or esmm or estmm or esfk" > gpurun_out/pytest_fd.log 2>&1
echo "exit $?" >> gpurun_out/pytest_fd.log
for i in 1 2 3; do
HXM_LIB=$PWD/ab/libhexamoe_fd0.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_fd0_$i.json 2>gpurun_out/bench_fd0_$i.err
HXM_LIB=$PWD/ab/libhexamoe_fd1.so timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_fd1_$i.json 2>gpurun_out/bench_fd1_$i.err
done
