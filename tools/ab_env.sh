# A/B an environment switch on the same box: bash tools/ab_env.sh "HXM_X=0" [bench args]
sw=$1; shift
for i in 1 2 3; do
  echo "A default"; python bench.py --no-cpu-baseline --steps 30 "$@" | python tools/summ.py 2>/dev/null | head -1
  echo "B $sw"; env $sw python bench.py --no-cpu-baseline --steps 30 "$@" | python tools/summ.py 2>/dev/null | head -1
done
