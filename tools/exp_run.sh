# usage: source tools/exp_run.sh; run [bench args]  -- per-kernel table (experiments only)
run() { echo "== $*"; timeout 300 python bench.py --no-cpu-baseline --steps 20 "$@" | python tools/summ.py; }
