# cluster tick kernel: stream GPU tests, config-4 section fused vs separate
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py -q -x -rf > gpurun_out/pytest_stream.log 2>&1; echo pytest=$?
tail -8 gpurun_out/pytest_stream.log
S="--no-cpu --no-mc --no-rc --no-e2e --no-config1 --no-server --steps 5"
for m in fused separate; do
  X=""; [ $m = separate ] && X="--stream-separate"
  timeout 600 python bench.py $S $X > gpurun_out/st_$m.json 2> gpurun_out/st_$m.err; echo $m=$?
  tail -3 gpurun_out/st_$m.err
done
python - <<'P'
import json
for n in ("fused", "separate"):
    try:
        D = json.loads(open(f"gpurun_out/st_{n}.json").read().splitlines()[-1])
        d = D["stream"]
        print(n, {k: d.get(k) for k in ("value", "ms_per_tick", "ok", "gpu_launches", "error", "parity_bad_clients")}, d.get("tick_only"))
    except Exception as e:
        print(n, "FAILED", e)
P
