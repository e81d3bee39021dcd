# A/B the config-4 tick: in-tree library vs build/ab/lib_head.so on the same box (experiments)
for i in 1 2 3; do
  for lib in build/ab/lib_head.so default; do
    if [ $lib = default ]; then unset VSB_LIB; else export VSB_LIB=$lib; fi
    echo "$lib $(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --live 1000000 --batch-log2 16 --no-mc --no-rc 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read())['stream']; print(round(d['value']), round(d['ms_per_tick'],4), d['ok'])")"
  done
done
