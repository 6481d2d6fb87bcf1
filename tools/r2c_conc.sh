set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "layer" > gpurun_out/pytest_conc.log 2>&1
echo "exit $?" >> gpurun_out/pytest_conc.log
HXM_BWD_CONC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "layer" >> gpurun_out/pytest_conc.log 2>&1
echo "exit $?" >> gpurun_out/pytest_conc.log
for i in 1 2 3; do
HXM_BWD_CONC=0 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_cc0_$i.json 2>gpurun_out/bench_cc0_$i.err
HXM_BWD_CONC=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_cc1_$i.json 2>gpurun_out/bench_cc1_$i.err
done
