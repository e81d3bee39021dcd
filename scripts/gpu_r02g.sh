# fused small fan-out: stream GPU tests, config-4 section eager vs graph; k_post without the FRESH clear (measurement)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_shim_gpu.py -q -x -rf > gpurun_out/pytest_stream.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_stream.log
S="--no-cpu --no-mc --no-rc --no-e2e --no-config1 --steps 5"
timeout 600 python bench.py $S > gpurun_out/st_graph.json 2> gpurun_out/st_graph.err; echo graph=$?
tail -3 gpurun_out/st_graph.err
timeout 600 python bench.py $S --stream-eager > gpurun_out/st_eager.json 2> gpurun_out/st_eager.err; echo eager=$?
python - <<'P'
import json
for n in ("graph", "eager"):
    try:
        D = json.loads(open(f"gpurun_out/st_{n}.json").read().splitlines()[-1])
        d = D["stream"]
        print(n, {k: d.get(k) for k in ("value", "ms_per_tick", "ok", "gpu_launches", "error")}, d.get("tick_only"), d.get("roofline", {}).get("kernel_ms"))
        v = D["server"]; print("  server", {k: v.get(k) for k in ("value", "ms_per_tick", "ok", "gpu_launches", "host_ms_per_tick", "error")})
    except Exception as e:
        print(n, "FAILED", e)
P
timeout 600 python scripts/ab.py --rounds 2 --section hash build/ab/lib_head.so build/ab/lib_nofresh.so 2>&1 | tee gpurun_out/ab_nofresh.txt
timeout 300 python scripts/single_time.py
