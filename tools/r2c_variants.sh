# the opt-in / fallback configurations over the parity suites
set -x
HXM_CHAIN=1 HXM_CHAIN_BWD=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py tests/test_gpu_chain.py -q > gpurun_out/pytest_var_chain.log 2>&1
echo "exit $?" >> gpurun_out/pytest_var_chain.log
HXM_CTA_PAIR=0 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q > gpurun_out/pytest_var_nopair.log 2>&1
echo "exit $?" >> gpurun_out/pytest_var_nopair.log
HXM_WIDE=0 HXM_WIDE_EST=0 HXM_PDL=0 HXM_SIDE=0 timeout 1500 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/pytest_var_plain.log 2>&1
echo "exit $?" >> gpurun_out/pytest_var_plain.log
