"""Experiment: does k_apply gain from warps whose ops all take the same path?
Config-2 batches permuted so that every group of G consecutive ops is
homogeneous by class, groups in random order: 'mut' = mutating (fresh
insert or erase) vs not, 'kind' = by op code only (what a pre-lookup
partition could do).  Times the apply pair (k_apply + k_post)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_1805_03709_b200 import BlockHashSet, workloads

dev = torch.device("cuda", 0)
spec = workloads.MixSpec(live=10_000_000, batch=1 << 22)
s = BlockHashSet(spec.bucket_count, spec.excess, device=dev)
for a in range(0, spec.live, 1 << 22):
    s.insert_keys(workloads.id_to_key_torch(torch.arange(a, min(spec.live, a + (1 << 22)), device=dev)))
torch.cuda.synchronize()
gen = torch.Generator(device=dev)
gen.manual_seed(7)
lo, hi = 0, spec.live


def homog(cls, G):
    """permutation: ops grouped by class into runs of G, runs shuffled."""
    groups = []
    for c in torch.unique(cls):
        idx = torch.nonzero(cls == c).flatten()
        idx = idx[torch.randperm(idx.numel(), device=dev, generator=gen)]
        pad = (-idx.numel()) % G
        groups += list(torch.split(idx, G))
    order = torch.randperm(len(groups), generator=torch.Generator().manual_seed(1)).tolist()
    return torch.cat([groups[i] for i in order])


modes = ["random", ("mut", 32), ("mut", 128), ("kind", 32), ("kind", 128)]
res = {str(m): [] for m in modes}
ok = True
for rep in range(7):
    for m in modes:
        ids, ops, expect = workloads.mix_batch_ids(spec, rep * len(modes) + modes.index(m), lo, hi, gen, dev)
        keys = workloads.id_to_key_torch(ids)
        if m != "random":
            kind, G = m
            if kind == "mut":
                cls = (((ops == 0) & (expect == 1)) | (ops == 2)).to(torch.int64)
            else:
                cls = ops.to(torch.int64)
            perm = homog(cls, G)
            keys, ops, expect = keys[perm].contiguous(), ops[perm].contiguous(), expect[perm].contiguous()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r, _ = s.apply(keys, ops)
        e1.record()
        torch.cuda.synchronize()
        ok &= bool(torch.equal(r, expect))
        if rep > 0:
            res[str(m)].append(e0.elapsed_time(e1))
        lo += spec.counts["erase"]
        hi += spec.counts["fresh"]
print(f"ok={ok}")
for m in modes:
    v = sorted(res[str(m)])
    print(f"  {str(m):>14}: {sum(v) / len(v):.4f} ms per apply pair (min {v[0]:.4f})")
