"""Experiment: k_apply on batches pre-ordered by bucket region (coarse
counting order: ops grouped into R regions of the bucket range, random
within a region) vs the random order, on the config-2 table and the
config-5 slice.  Times the apply launch pair (k_apply + k_post) with CUDA
events; results are in permuted order (timing only; the per-op results are
still checked against the permuted expectation).
Usage: python scripts/sorted_apply_exp.py [live] [batch_log2]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_1805_03709_b200 import BlockHashSet, hash_keys, workloads

dev = torch.device("cuda", 0)
live = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
blog = int(sys.argv[2]) if len(sys.argv) > 2 else 22
spec = workloads.MixSpec(live=live, batch=1 << blog)
s = BlockHashSet(spec.bucket_count, spec.excess, device=dev)
for a in range(0, spec.live, 1 << 22):
    s.insert_keys(workloads.id_to_key_torch(torch.arange(a, min(spec.live, a + (1 << 22)), device=dev)))
torch.cuda.synchronize()
gen = torch.Generator(device=dev)
gen.manual_seed(5)
lo, hi = 0, spec.live
modes = ["random", 16, 64, 256, 1024, 4096]
steps_per_mode = 6
res = {m: [] for m in modes}
ok = True
for rep in range(steps_per_mode):
    for m in modes:
        ids, ops, expect = workloads.mix_batch_ids(spec, rep * len(modes) + modes.index(m), lo, hi, gen, dev)
        keys = workloads.id_to_key_torch(ids)
        if m != "random":
            b = hash_keys(keys, spec.bucket_count)
            region = b * m // spec.bucket_count
            perm = torch.argsort(region * (1 << 32) + torch.randint(0, 1 << 30, region.shape, device=dev,
                                                                    generator=gen))
            keys, ops, expect = keys[perm].contiguous(), ops[perm].contiguous(), expect[perm].contiguous()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r, _ = s.apply(keys, ops)
        e1.record()
        torch.cuda.synchronize()
        ok &= bool(torch.equal(r, expect))
        if rep > 0:
            res[m].append(e0.elapsed_time(e1))
        lo += spec.counts["erase"]
        hi += spec.counts["fresh"]
print(f"live={live} batch=2^{blog} ok={ok}")
for m in modes:
    v = sorted(res[m])
    print(f"  order {str(m):>7}: {sum(v) / len(v):.4f} ms per apply (min {v[0]:.4f})  "
          f"{spec.batch / (sum(v) / len(v)) / 1e6:.2f} G ops/s")
