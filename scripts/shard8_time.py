"""An 8-rank node simulated on one GPU (OneGpuShardGroup): config-2 per-rank
tables (10M keys) and 2^22-op batches routed through the peer windows.  The
whole node's work runs on one GPU, so ms/batch here ~ 8x a real rank's; the
per-kernel times (ncu) show the G=8 routing costs.  Usage:
python scripts/shard8_time.py [steps] [world]"""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # one hardware queue per rank stream
sys.path.insert(0, os.getcwd())
import torch

from paper_1805_03709_b200 import BlockHashSet, workloads
from paper_1805_03709_b200.shard import OneGpuShardGroup

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = torch.device("cuda", 0)
spec = workloads.MixSpec()
tabs = [BlockHashSet(spec.bucket_count, spec.excess, device=dev) for _ in range(world)]
g = OneGpuShardGroup(tabs, max_batch=spec.batch)
z = lambda n: torch.zeros(n, dtype=torch.uint8, device=dev)  # noqa: E731
for a in range(0, spec.live, spec.batch):
    b = min(spec.live, a + spec.batch)
    g.apply([workloads.id_to_key_torch(torch.arange((r << 40) + a, (r << 40) + b, device=dev)) for r in range(world)],
            [z(b - a)] * world)
torch.cuda.synchronize()
gens = [torch.Generator(device=dev) for _ in range(world)]
for r, gg in enumerate(gens):
    gg.manual_seed(r)
lo = [r << 40 for r in range(world)]
hi = [(r << 40) + spec.live for r in range(world)]
batches = []
for step in range(steps + 2):
    ks, os_, ex = [], [], []
    for r in range(world):
        ids, ops, expect = workloads.mix_batch_ids(spec, step, lo[r], hi[r], gens[r], dev)
        ids = torch.where(ids >= workloads.MISS_BASE, ids + (r << 50), ids)
        ks.append(workloads.id_to_key_torch(ids))
        os_.append(ops)
        ex.append(expect)
        lo[r] += spec.counts["erase"]
        hi[r] += spec.counts["fresh"]
    batches.append((ks, os_, ex))
ok = True
for bi, (ks, os_, ex) in enumerate(batches[:2]):
    out = g.apply(ks, os_)
    torch.cuda.synchronize()
    for r, (o, e) in enumerate(zip(out, ex)):
        bad = o != e
        if bool(bad.any()):
            ok = False
            kinds = os_[r][bad]
            print(f"batch {bi} rank {r}: {int(bad.sum())} mismatches; ops {torch.bincount(kinds.long(), minlength=3).tolist()}"
                  f" got {torch.bincount(o[bad].long(), minlength=2).tolist()}", flush=True)
for t in tabs:
    try:
        t.check_capacity()
    except Exception as exc:  # noqa: BLE001
        print("capacity:", exc, flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
outs = [g.apply(ks, os_) for ks, os_, _ in batches[2:]]
e1.record()
torch.cuda.synchronize()
ok &= all(torch.equal(o, e) for out, (_, _, ex) in zip(outs, batches[2:]) for o, e in zip(out, ex))
ms = e0.elapsed_time(e1) / steps
print(f"world {world} on one GPU: {ms:.3f} ms per collective batch ({world} x {spec.batch} ops) "
      f"= {world * spec.batch / ms / 1e6:.2f} G ops/s on this GPU; ok={ok}", flush=True)
g.check()
