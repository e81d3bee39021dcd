# functional check of the N>1 bench path (config-5 defaults: 1e9/N keys per rank, 2^24-op batches)
# with both ranks on one GPU over gloo (numbers not meaningful; the route and sizing are)
mkdir -p gpurun_out
VSB_BENCH_ONE_GPU=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2=$?
tail -5 gpurun_out/bench_n2.err
grep -c "NCCL INFO" gpurun_out/bench_n2.err
python - <<'P'
import json
d = json.loads(open("gpurun_out/bench_n2.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value", "n_gpus", "ms_per_step", "parity_ok", "gpu_launches")}, d["config"]["workload"], d["config"].get("exchange"))
print("mc", {k: (d.get("mc") or {}).get(k) for k in ("value", "ok", "error")})
P
nvidia-smi --query-gpu=memory.used --format=csv
