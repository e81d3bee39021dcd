# build MC kernel variants on the box and time each (experiments)
timeout 300 python -m pytest tests/test_mc_gpu.py -q -x 2>&1 | tail -1
for v in "VSB_MC_MINBLOCKS=1" "VSB_MC_MINBLOCKS=8" "VSB_MC_MINBLOCKS=10" "VSB_MC_MINBLOCKS=12" "VSB_MC_STAGES=3 VSB_MC_MINBLOCKS=8"; do
  name=$(echo $v | tr ' =' '__')
  python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_$name.so', defines=tuple('$v'.split()))" && \
  VSB_LIB=/tmp/lib_$name.so timeout 300 python scripts/mc_time.py 2>&1 | tail -1
done
