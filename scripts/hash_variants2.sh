# hash op-kernel variants (experiments): build each -D set on the box, time config 2 (bench hash section)
for v in "VSB_HASH_STRIPES=128"; do
  name=$(echo $v | tr ' =' '__')
  python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_$name.so', defines=tuple('$v'.split()))" && \
  VSB_LIB=/tmp/lib_$name.so timeout 600 python bench.py --no-cpu --no-mc --no-stream --no-rc --no-e2e --steps 200 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4), d['parity_ok'])"
done
