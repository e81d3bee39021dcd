"""vs_table_probe_sol (1 dependent random 16-B load per op, 2^22 ops) on a
256 MiB and a 4 GiB table, for an ncu capture of both launches (L2 hit rate,
DRAM sectors, ops/s): where the 3x drop of the random-access rate comes from."""
import ctypes
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
for lg in (24, 28):
    s = BlockHashSet(1 << (lg - 1), 1 << (lg - 1), device=dev)
    for _ in range(3):
        lib.vs_table_probe_sol(s.handle, B, 1, _lib.ptr(out), st)
    torch.cuda.synchronize()
    del s
    torch.cuda.empty_cache()
