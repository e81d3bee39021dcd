# A/B the in-tree hash kernels against build/ab/lib_head.so on the same box (experiments)
for i in 1 2; do
  for lib in build/ab/lib_head.so default; do
    if [ $lib = default ]; then unset VSB_LIB; else export VSB_LIB=$lib; fi
    echo "$lib $(timeout 300 python bench.py --no-cpu --no-mc --no-stream --no-rc --no-e2e --steps 300 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4), d['parity_ok'])")"
  done
done
