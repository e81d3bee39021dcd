"""torch.profiler kernel table of the RC fusion loop (experiments)."""
import os, sys, types
sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1805_03709_b200 import workloads
from paper_1805_03709_b200.voxel_model import GpuVoxelModel

depth, color, Rs, ts, (fx, fy, cx, cy, w, h) = workloads.room_frames(12, 640, 480)
intr = types.SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)
cfg = types.SimpleNamespace(voxel_size=0.005, truncation=0.06, max_weight=128.0, alloc_stride=1)
dev = torch.device("cuda", 0)
m = GpuVoxelModel(cfg, bucket_count=1 << 21, excess_capacity=1 << 21, device=dev)
dd = torch.from_numpy(depth).to(dev)
cc = torch.from_numpy(color).to(dev)
for f in range(7):
    m.allocate_blocks_tensor(dd[f], (Rs[f], ts[f]), intr)
    m.integrate_frame_tensor(dd[f], cc[f], (Rs[f], ts[f]), intr)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as p:
    for f in range(7, 12):
        m.allocate_blocks_tensor(dd[f], (Rs[f], ts[f]), intr)
        m.integrate_frame_tensor(dd[f], cc[f], (Rs[f], ts[f]), intr)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=22, max_name_column_width=40))
