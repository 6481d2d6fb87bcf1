set -x
for i in 1 2; do
for sw in "X=0" "HXM_REVERSE=0" "HXM_L2HINT=0" "HXM_PRO_BLOCKS=1" "HXM_WIDE=0"; do
tag=$(echo $sw | tr '=' '_')
env $sw timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/bench_k_${tag}_$i.json 2>/dev/null
done
done
