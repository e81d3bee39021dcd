"""Host cost of GpuServerCore.on_tsdf_batch(sync=False) per tick, split into
the Python wrapper and the vs_server_tick C call (cProfile over 200 ticks
while the GPU is kept busy far ahead, so no call waits on the device)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_1805_03709_b200 import GpuServerCore, workloads

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
T = 85
upd = torch.from_numpy(scene_np[rng.integers(0, len(scene_np), (T, 512))]).to(dev)
rows = torch.stack([workloads.room_tsdf_rows(upd[t]) for t in range(T)])
torch.cuda.synchronize()
for t in range(5):
    core.on_tsdf_batch(upd[t], rows[t], sync=False)
torch.cuda.synchronize()
torch.cuda._sleep(200_000_000)  # keep the GPU busy (~0.1 s): 40 ticks stay within the launch queue
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()  # after the sleep kernel: the ticks below are all queued when it ends
t0 = time.perf_counter()
for t in range(5, T // 2):
    core.on_tsdf_batch(upd[t], rows[t], sync=False)
dt = (time.perf_counter() - t0) / (T // 2 - 5)
e1.record()
torch.cuda.synchronize()
print(f"host per tick (no profiler): {dt * 1e6:.1f} us; device per tick, queued back to back: "
      f"{e0.elapsed_time(e1) * 1e3 / (T // 2 - 5):.1f} us")
torch.cuda._sleep(200_000_000)
pr = cProfile.Profile()
pr.enable()
for t in range(T // 2, T):
    core.on_tsdf_batch(upd[t], rows[t], sync=False)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
