"""Random-access speed of light vs table size (the probe
falls ~3x at the 2.9 GB config-5 slice).  vs_table_probe_sol: 1..2 dependent
random 16-B entry loads per op over a table of C slots (16 B each), 2^22
ops, k_apply's launch shape.  The knee locates the reach of the GPU's
address-translation caches.  Usage: python scripts/sol_sizes.py"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_1805_03709_b200 import BlockHashSet, _lib

dev = torch.device("cuda", 0)
lib = _lib.load()
B = 1 << 22
out = torch.empty(B, dtype=torch.uint8, device=dev)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {}
for lg in range(20, 31):
    cap = 1 << lg
    s = BlockHashSet(cap // 2, cap // 2, device=dev)
    row = {}
    for hops in (1, 2):
        for _ in range(3):
            lib.vs_table_probe_sol(s.handle, B, hops, _lib.ptr(out), st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            lib.vs_table_probe_sol(s.handle, B, hops, _lib.ptr(out), st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        row[hops] = hops * B / ms / 1e6
    res[f"{cap * 16 / 2**20:.0f} MiB"] = row
    print(f"table {cap * 16 / 2**20:8.0f} MiB: {row[1]:6.1f} / {row[2]:6.1f} G dependent loads/s (1 / 2 hops)",
          flush=True)
    del s
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/sol_sizes.json", "w"), indent=1)
