# RC fusion frames with and without programmatic dependent launches (experiments)
python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_nopdl.so', defines=('VSB_PDL=0',))"
for i in 1 2 3; do
  for lib in default /tmp/lib_nopdl.so; do
    if [ $lib = default ]; then unset VSB_LIB; else export VSB_LIB=$lib; fi
    echo "$lib $(timeout 300 python bench.py --no-cpu --no-mc --no-stream --no-e2e --steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read())['rc']; print(round(d['value']), round(d['ms_per_frame'],4), d.get('ok'), round(d.get('value_sync_api',0)))")"
  done
done
unset VSB_LIB
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
