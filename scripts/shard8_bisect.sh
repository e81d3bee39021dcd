# bisect the intermittent 8-rank simulation mismatch across hash fast paths (debug)
for v in "VSB_AB=0"; do
  name=$(echo $v | tr ' =' '__')
  python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_$name.so', defines=tuple('$v'.split()))"
  for i in 1 2 3 4 5; do echo "$v $(VSB_LIB=/tmp/lib_$name.so timeout 300 python scripts/shard8_time.py 10 8 2>&1 | tail -1)"; done
done
