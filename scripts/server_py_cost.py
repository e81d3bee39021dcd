"""Python-wrapper share of GpuServerCore.on_tsdf_batch(sync=False): the same
loop with vs_server_tick replaced by a no-op (experiments)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_1805_03709_b200 import GpuServerCore, _lib, workloads

dev = torch.device("cuda", 0)
scene_np = workloads.room_block_keys()[:200_000]
scene = torch.from_numpy(scene_np).to(dev)
core = GpuServerCore(1 << 19, 1 << 19, stream_buckets=1 << 19, stream_excess=1 << 19, max_batch=1 << 16, device=dev)
for a in range(0, len(scene), 1 << 16):
    k = scene[a:a + (1 << 16)]
    core.on_tsdf_batch(k, workloads.room_tsdf_rows(k), sync=False)
for c in range(16):
    core.attach(bytes([c]) * 16)
rng = np.random.default_rng(1)
T = 60
upd = torch.from_numpy(scene_np[rng.integers(0, len(scene_np), (T, 512))]).to(dev)
rows = torch.stack([workloads.room_tsdf_rows(upd[t]) for t in range(T)])
torch.cuda.synchronize()


def run():
    torch.cuda._sleep(100_000_000)
    t0 = time.perf_counter()
    for t in range(10, T):
        core.on_tsdf_batch(upd[t], rows[t], sync=False)
    dt = (time.perf_counter() - t0) / (T - 10)
    torch.cuda.synchronize()
    return dt * 1e6


full = [run() for _ in range(3)]
lib = _lib.load()
real = lib.vs_server_tick
try:
    lib.vs_server_tick = lambda *a: 0
    py = [run() for _ in range(3)]
finally:
    lib.vs_server_tick = real
print(f"host us per tick: full {min(full):.1f}, python wrapper only {min(py):.1f}")
