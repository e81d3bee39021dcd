"""Time the RC fusion loop alone (experiments; the contract bench is bench.py)."""
import json, os, sys, types
sys.path.insert(0, os.getcwd())
import torch
from paper_1805_03709_b200 import _lib, workloads
from paper_1805_03709_b200.voxel_model import GpuVoxelModel

n = int(os.environ.get("RC_FRAMES", "20"))
dev = torch.device("cuda", 0)
depth, color, Rs, ts, (fx, fy, cx, cy, w, h) = workloads.room_frames(n + 2, 640, 480)
intr = types.SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)
cfg = types.SimpleNamespace(voxel_size=0.005, truncation=0.06, max_weight=128.0, alloc_stride=1)
model = GpuVoxelModel(cfg, bucket_count=1 << 21, excess_capacity=1 << 21, device=dev)
dd = torch.from_numpy(depth).to(dev)
cc = torch.from_numpy(color).to(dev)
for f in range(2):
    model.allocate_blocks_tensor(dd[f], (Rs[f], ts[f]), intr)
    model.integrate_frame_tensor(dd[f], cc[f], (Rs[f], ts[f]), intr)
torch.cuda.synchronize()
ea, eb = [], []
tot = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot[0].record()
for f in range(2, n + 2):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    model.allocate_blocks_tensor(dd[f], (Rs[f], ts[f]), intr)
    e[1].record()
    model.integrate_frame_tensor(dd[f], cc[f], (Rs[f], ts[f]), intr)
    e[2].record()
    ea.append(e)
tot[1].record()
torch.cuda.synchronize()
alloc = sum(e[0].elapsed_time(e[1]) for e in ea) / n
integ = sum(e[1].elapsed_time(e[2]) for e in ea) / n
print(json.dumps({"ms_per_frame": tot[0].elapsed_time(tot[1]) / n, "alloc_ms": alloc, "integrate_ms": integ,
                  "blocks": model.blocks.approx_size()}), flush=True)
