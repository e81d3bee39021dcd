# MC encoder variants (experiments): build each on the box, time config 3
for v in "VSB_MC_STAGES=2" "VSB_MC_MINBLOCKS_KEYS=12 VSB_MC_MINBLOCKS_NBR=10"; do
  name=$(echo $v | tr ' =' '__')
  python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_$name.so', defines=tuple('$v'.split()))" && \
  echo "$v $(VSB_LIB=/tmp/lib_$name.so timeout 600 python scripts/mc_time.py 2>&1 | tail -1)"
done
