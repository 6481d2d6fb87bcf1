# A/B two in-tree builds on the same box: bash tools/ab.sh ab/old.so ab/new.so [bench args]
a=$1; b=$2; shift 2
for i in 1 2 3; do
  echo "A $a"; HXM_LIB=$PWD/$a python bench.py --no-cpu-baseline --steps 30 "$@" | python tools/summ.py 2>/dev/null | head -1
  echo "B $b"; HXM_LIB=$PWD/$b python bench.py --no-cpu-baseline --steps 30 "$@" | python tools/summ.py 2>/dev/null | head -1
done
