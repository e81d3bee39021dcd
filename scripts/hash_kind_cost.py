"""Per-op-kind cost of one config-2 mixed batch (experiment).

Each variant builds a fresh 10M-key table, applies one untimed mixed batch,
then times ONE batch generated from the same state with some op kinds turned
into finds of the same keys (so every variant sees the same table and the
same keys; only the op codes differ).  Times apply + post with CUDA events
on the launching stream; 3 fresh tables per variant, median reported.
Marginal cost of a kind = T(with it) - T(with it turned into finds)."""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_1805_03709_b200 import BlockHashSet, workloads

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
spec = workloads.MixSpec()
c = spec.counts
F, P, H, M, E = c["fresh"], c["present"], c["hit"], c["miss"], c["erase"]


def one(transform, seed):
    s = BlockHashSet(spec.bucket_count, spec.excess, device=dev)
    for a in range(0, spec.live, 1 << 22):
        s.insert_keys(workloads.id_to_key_torch(torch.arange(a, min(spec.live, a + (1 << 22)), device=dev)))
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    ids, ops, _ = workloads.mix_batch_ids(spec, 0, 0, spec.live, gen, dev)
    s.apply(workloads.id_to_key_torch(ids), ops)
    ids, ops, expect = workloads.mix_batch_ids(spec, 1, E, spec.live + F, gen, dev)
    keys = workloads.id_to_key_torch(ids)
    ops = transform(ops, expect).contiguous()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s.apply(keys, ops)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    del s
    torch.cuda.empty_cache()
    return ms


FIND = lambda o: torch.ones_like(o)
fresh = lambda o, e: (o == 0) & (e == 1)
present = lambda o, e: (o == 0) & (e == 0)
erase = lambda o, e: o == 2
variants = [
    ("mix 50/30/20 (as the bench)", lambda o, e: o),
    ("erases -> finds", lambda o, e: torch.where(erase(o, e), FIND(o), o)),
    ("fresh inserts -> finds", lambda o, e: torch.where(fresh(o, e), FIND(o), o)),
    ("fresh inserts + erases -> finds", lambda o, e: torch.where(fresh(o, e) | erase(o, e), FIND(o), o)),
    ("all finds (same keys)", lambda o, e: FIND(o)),
]
res = {}
for label, t in variants:
    ts = [one(t, 11 + r) for r in range(3)]
    res[label] = statistics.median(ts)
    print(f"{label:36s} {res[label] * 1e3:7.1f} us  ({', '.join(f'{x * 1e3:.1f}' for x in ts)})", flush=True)
m = [res[l] for l, _ in variants]
print(f"marginal per 838,861 fresh inserts : {(m[1] - m[3]) * 1e3:6.1f} us  (mix - fresh->find: {(m[0] - m[2]) * 1e3:.1f})")
print(f"marginal per 838,861 erases        : {(m[2] - m[3]) * 1e3:6.1f} us  (mix - erase->find: {(m[0] - m[1]) * 1e3:.1f})")
print(f"marginal per 1,258,291 present ins.: {(m[3] - m[4]) * 1e3:6.1f} us")
print(f"all {spec.batch:,} ops as finds    : {m[4] * 1e3:6.1f} us")
