# stream section (config 4) across unlock / PDL build variants, interleaved (experiments)
python -c "
import sys; sys.path.insert(0,'.'); from paper_1805_03709_b200 import build
build.build(out='/tmp/lib_x.so', defines=('VSB_HASH_ST_UNLOCK=0',))
build.build(out='/tmp/lib_np.so', defines=('VSB_PDL=0',))
build.build(out='/tmp/lib_old.so', defines=('VSB_HASH_ST_UNLOCK=0','VSB_PDL=0'))"
for i in 1 2 3; do
  for lib in default /tmp/lib_x.so /tmp/lib_np.so /tmp/lib_old.so; do
    if [ $lib = default ]; then unset VSB_LIB; else export VSB_LIB=$lib; fi
    echo "$lib $(timeout 300 python bench.py --no-cpu --no-mc --no-rc --no-e2e --steps 50 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read())['stream']; print(round(d['value']), round(d['ms_per_tick'],4), round(d['fill_16_clients_ms'],2), d['ok'])")"
  done
done
