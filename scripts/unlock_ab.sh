# A/B the bucket-unlock flavour (exchange vs store) and predecessor validation on one box (experiments)
python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_st.so', defines=('VSB_HASH_ST_UNLOCK=1',)); build.build(out='/tmp/lib_stv.so', defines=('VSB_HASH_ST_UNLOCK=1','VSB_HASH_VALIDATE_PREV=1'))"
for i in 1 2 3; do
  for lib in default /tmp/lib_st.so /tmp/lib_stv.so; do
    if [ $lib = default ]; then unset VSB_LIB; else export VSB_LIB=$lib; fi
    echo "$lib $(timeout 300 python bench.py --no-cpu --no-mc --no-stream --no-rc --no-e2e --steps 300 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4), d['parity_ok'])")"
  done
done
for lib in /tmp/lib_st.so /tmp/lib_stv.so; do
  for i in 1 2 3 4 5; do echo "$lib $(VSB_LIB=$lib timeout 300 python scripts/shard8_time.py 10 8 2>&1 | tail -1)"; done
done
VSB_LIB=/tmp/lib_st.so timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
