"""Dependent random-access speed of light on the config-2 table storage:
vs_table_probe_sol with 1..4 dependent 16-B entry loads per op, k_apply's
launch shape, against k_apply itself on the same table.  Usage:
python scripts/sol_probe.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_1805_03709_b200 import BlockHashSet, _lib, workloads

dev = torch.device("cuda", 0)
spec = workloads.MixSpec()
s = BlockHashSet(spec.bucket_count, spec.excess, device=dev)
for a in range(0, spec.live, 1 << 22):
    s.insert_keys(workloads.id_to_key_torch(torch.arange(a, min(spec.live, a + (1 << 22)), device=dev)))
B = spec.batch
out = torch.empty(B, dtype=torch.uint8, device=dev)
lib = _lib.load()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {}
for hops in (1, 2, 3, 4, 6):
    for _ in range(3):
        lib.vs_table_probe_sol(s.handle, B, hops, _lib.ptr(out), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        lib.vs_table_probe_sol(s.handle, B, hops, _lib.ptr(out), st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res[hops] = ms
    print(f"hops={hops}: {ms * 1e3:7.1f} us/launch  {B / ms / 1e6:6.2f} G ops/s  {hops * B / ms / 1e6:6.2f} G loads/s",
          flush=True)
gen = torch.Generator(device=dev)
gen.manual_seed(3)
lo, hi = 0, spec.live
bs = []
for step in range(23):
    ids, ops, expect = workloads.mix_batch_ids(spec, step, lo, hi, gen, dev)
    bs.append((workloads.id_to_key_torch(ids), ops))
    lo += spec.counts["erase"]
    hi += spec.counts["fresh"]
for k, o in bs[:3]:
    s.apply(k, o)
with _lib.Profile() as prof:
    for k, o in bs[3:]:
        s.apply(k, o)
ms = prof.ms["hash"] / prof.count["hash"]
print(f"k_apply: {ms * 1e3:7.1f} us/launch  {B / ms / 1e6:6.2f} G ops/s")
