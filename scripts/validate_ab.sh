python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_v.so', defines=('VSB_HASH_VALIDATE_PREV=1',))"
for i in 1 2 3; do
  for lib in /tmp/lib_v.so default; do
    if [ $lib = default ]; then unset VSB_LIB; else export VSB_LIB=$lib; fi
    echo "$lib $(timeout 300 python bench.py --no-cpu --no-mc --no-stream --no-rc --no-e2e --steps 300 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4), d['parity_ok'])")"
  done
done
unset VSB_LIB
VARIANTS="VSB_HASH_VALIDATE_PREV=1" RUNS=10 bash scripts/shard8_bisect.sh
