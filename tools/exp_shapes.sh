# per-kernel timing sweep (bench lines are experiments, not the headline)
run() { echo "== $*"; timeout 300 python bench.py --no-cpu-baseline --steps 20 "$@" | python -c "
import json,sys
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print('ms %.3f tok/s %.1fM' % (d['ms_per_step'], d['value']/1e6))
    for k,v in d['kernels'].items(): print('  %-14s %7.1f us %7.1f %s %.2f' % (k, v['avg_us'], v['achieved'], v['unit'], v['frac']))
"; }
run
HXM_CTA_PAIR=0 run
run --shape 32,2,384,1536,65536
run --shape 32,2,1024,1536,16384
run --shape 32,2,384,4096,16384
run --shape 32,2,768,1536,16384
