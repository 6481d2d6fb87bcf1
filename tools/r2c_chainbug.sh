set -x
HXM_LIB=$PWD/ab/libhexamoe_chainbug.so HXM_CHAIN=1 HXM_CHAIN_BWD=1 HXM_CHAIN_FPT=0 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tests/_chain_worker.py /tmp/x.pt > gpurun_out/chainbug_memcheck.log 2>&1
echo "exit $?" >> gpurun_out/chainbug_memcheck.log
for f in 0 1; do
HXM_LIB=$PWD/ab/libhexamoe_chainbug.so HXM_CHAIN=1 HXM_CHAIN_BWD=0 HXM_CHAIN_FPT=$f timeout 300 python tests/_chain_worker.py /tmp/x.pt > gpurun_out/chainbug_fwd_$f.log 2>&1; echo "fwd fpt=$f exit $?" >> gpurun_out/chainbug_fwd_$f.log
HXM_LIB=$PWD/ab/libhexamoe_chainbug.so HXM_CHAIN=0 HXM_CHAIN_BWD=1 HXM_CHAIN_FPT=$f timeout 300 python tests/_chain_worker.py /tmp/x.pt > gpurun_out/chainbug_bwd_$f.log 2>&1; echo "bwd fpt=$f exit $?" >> gpurun_out/chainbug_bwd_$f.log
done
