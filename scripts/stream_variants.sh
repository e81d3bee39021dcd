# stream-set extraction CTA shape variants (experiments): config-4 tick timing
for v in "VSB_EXTRACT_THREADS=256" "VSB_EXTRACT_THREADS=512 VSB_EXTRACT_K=4" "VSB_EXTRACT_THREADS=1024 VSB_EXTRACT_K=2" "VSB_EXTRACT_THREADS=1024 VSB_EXTRACT_K=4"; do
  name=$(echo $v | tr ' =' '__')
  python -c "import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build; build.build(out='/tmp/lib_$name.so', defines=tuple('$v'.split()))" && \
  echo "$v $(VSB_LIB=/tmp/lib_$name.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --live 1000000 --batch-log2 16 --no-mc --no-rc 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read())['stream']; print(round(d['value']), round(d['ms_per_tick'],4), d['ok'])")"
done
