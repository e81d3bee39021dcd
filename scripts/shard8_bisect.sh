# 8-rank simulation stress across hash build variants (debug): VARIANTS="A=1 B=0;C=1" RUNS=5
IFS=';' read -ra vs <<< "${VARIANTS:-VSB_AB=0}"
for v in "${vs[@]}"; do
  name=$(echo $v | tr ' =' '__')
  python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_$name.so', defines=tuple('$v'.split()))"
  for i in $(seq ${RUNS:-5}); do echo "$v $(VSB_LIB=/tmp/lib_$name.so timeout 300 python scripts/shard8_time.py 10 8 2>&1 | tail -1)"; done
done
