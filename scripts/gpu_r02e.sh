# L2 fetch granularity vs the random entry accesses of k_apply (HEAD design)
mkdir -p gpurun_out
A="--no-cpu --no-mc --no-stream --no-rc --no-e2e --no-server --no-config1 --steps 200"
for g in "" 32 64 128; do
  VSB_L2_FETCH=$g python scripts/l2fetch_probe.py 2>&1 | tail -1
  VSB_L2_FETCH=$g timeout 300 python bench.py $A > gpurun_out/l2f_$g.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/l2f_$g.json').read().splitlines()[-1]); print('fetch=$g', round(d['value']), d['roofline']['kernel_ms'], d['parity_ok'])"
  VSB_L2_FETCH=$g timeout 300 python bench.py $A --config5-slice 8 --steps 10 > gpurun_out/l2f5_$g.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/l2f5_$g.json').read().splitlines()[-1]); print('c5 fetch=$g', round(d['value']), d['roofline']['kernel_ms'], d['parity_ok'])"
done
