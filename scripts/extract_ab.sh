# config-4 tick: extracted keys erased at scan time (default) vs after the cluster-wide write-out (experiments)
python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_old.so', defines=('VSB_EXTRACT_ERASE_AT_SCAN=0',))"
for i in 1 2 3; do
  for lib in default /tmp/lib_old.so; do
    if [ $lib = default ]; then unset VSB_LIB; else export VSB_LIB=$lib; fi
    echo "$lib $(timeout 300 python bench.py --no-cpu --no-mc --no-rc --no-e2e --steps 50 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read())['stream']; print(round(d['value']), round(d['ms_per_tick'],4), d['ok'], d['inserts'], d['removes'])")"
  done
done
unset VSB_LIB
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
