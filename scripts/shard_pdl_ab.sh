# peer-sharded route with and without programmatic dependent launches (experiments)
python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_nopdl.so', defines=('VSB_PDL=0',))"
timeout 600 python -m pytest tests/test_shard_gpu.py -q -x 2>&1 | tail -1
for i in 1 2; do
  echo "pdl   $(timeout 300 python scripts/shard_time.py 30 2>&1 | tail -2 | tr '\n' ' ')"
  echo "nopdl $(VSB_LIB=/tmp/lib_nopdl.so timeout 300 python scripts/shard_time.py 30 2>&1 | tail -2 | tr '\n' ' ')"
done
for i in 1 2 3; do echo "pdl8 $(timeout 300 python scripts/shard8_time.py 10 8 2>&1 | tail -1)"; done
