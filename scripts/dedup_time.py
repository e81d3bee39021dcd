"""k_dedup_small in isolation (experiments): the per-tick affected dedup of 512 updated room keys."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1805_03709_b200 import BlockHashSet, _lib, workloads
dev = torch.device("cuda", 0)
keys = torch.from_numpy(workloads.room_block_keys()).to(dev)
gen = torch.Generator(device=dev); gen.manual_seed(5)
upd = keys[torch.randint(0, keys.shape[0], (512,), generator=gen, device=dev)].contiguous()
scratch = BlockHashSet(1 << 14, 1 << 14, device=dev)
out = torch.empty((4096, 3), dtype=torch.int32, device=dev)
n = torch.empty(1, dtype=torch.int64, device=dev)
lib = _lib.load()
cs = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
for _ in range(5):
    lib.vs_affected_dedup(scratch.handle, _lib.ptr(upd), 512, _lib.ptr(out), _lib.ptr(n), cs)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    lib.vs_affected_dedup(scratch.handle, _lib.ptr(upd), 512, _lib.ptr(out), _lib.ptr(n), cs)
e1.record(); torch.cuda.synchronize()
print("dedup us/call (events, back-to-back):", round(e0.elapsed_time(e1) * 10, 2), "n =", int(n.item()))
