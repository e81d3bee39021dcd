# 8-rank simulation timing: store unlock (default) vs exchange unlock, interleaved (experiments)
python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_x.so', defines=('VSB_HASH_ST_UNLOCK=0',))"
for i in 1 2 3 4 5 6; do
  echo "st $(timeout 300 python scripts/shard8_time.py 10 8 2>&1 | tail -1)"
  echo "xchg $(VSB_LIB=/tmp/lib_x.so timeout 300 python scripts/shard8_time.py 10 8 2>&1 | tail -1)"
done
