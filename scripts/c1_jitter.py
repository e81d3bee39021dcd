"""Config-1 step timing jitter: wall vs host CPU time per loop of 200 steps (experiments)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1805_03709_b200 import BlockHashSet, workloads

dev = torch.device("cuda", 0)
keys, absent = workloads.config1_keys()
import numpy as np
dk = torch.from_numpy(keys).to(dev)
dp = torch.from_numpy(np.concatenate([keys, absent])).to(dev)
s = BlockHashSet(1 << 17, 1 << 17, device=dev)
if len(sys.argv) > 1:  # free a large allocation first (as the bench's earlier sections do)
    big = [torch.empty(1 << 30, dtype=torch.uint8, device=dev) for _ in range(int(sys.argv[1]))]
    for b in big:
        b.fill_(1)
    torch.cuda.synchronize()
    del big, b
    torch.cuda.empty_cache()
for rep in range(8):
    torch.cuda.synchronize()
    w0, c0 = time.perf_counter(), time.process_time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        s.insert_keys(dk); s.find_keys(dp); s.erase_keys(dk)
    e1.record()
    w1, c1 = time.perf_counter(), time.process_time()
    torch.cuda.synchronize()
    print(f"rep {rep}: gpu {e0.elapsed_time(e1) / 200 * 1e3:.0f} us/step, host wall {(w1 - w0) / 200 * 1e6:.0f} us/step, "
          f"host cpu {(c1 - c0) / 200 * 1e6:.0f} us/step, loadavg {os.getloadavg()[0]:.1f}, cpus {os.cpu_count()}", flush=True)
