"""Cost of the peer-window sharded path at world 1 (self window) against the
plain table on the config-2 mix: partition + push + routed apply + post +
return + waits, all on one GPU.  Also times each kernel of the batch with
the library profiler.  Usage: python scripts/shard_time.py [steps]"""
import os
import sys
import tempfile

sys.path.insert(0, os.getcwd())
import torch
import torch.distributed as dist

from paper_1805_03709_b200 import BlockHashSet, workloads
from paper_1805_03709_b200.shard import ShardedBlockHashSet

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
live = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
blog = int(sys.argv[3]) if len(sys.argv) > 3 else 22
dev = torch.device("cuda", 0)
dist.init_process_group("gloo", init_method=f"file://{tempfile.mkdtemp()}/pg", rank=0, world_size=1)
spec = workloads.MixSpec(live=live, load_factor=0.7, batch=1 << blog)
res = {}
for mode in ("table", "peer"):
    s = BlockHashSet(spec.bucket_count, spec.excess, device=dev)
    sh = ShardedBlockHashSet(s, exchange="peer", max_batch=spec.batch) if mode == "peer" else None
    for a in range(0, spec.live, 1 << 22):
        k = workloads.id_to_key_torch(torch.arange(a, min(spec.live, a + (1 << 22)), device=dev))
        s.insert_keys(k)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    lo, hi = 0, spec.live
    batches = []
    for step in range(steps + 3):
        ids, ops, expect = workloads.mix_batch_ids(spec, step, lo, hi, gen, dev)
        batches.append((workloads.id_to_key_torch(ids), ops, expect))
        lo += spec.counts["erase"]
        hi += spec.counts["fresh"]
    f = (lambda k, o: sh.apply(k, o)) if sh else (lambda k, o: s.apply(k, o)[0])
    ok = True
    for i in range(3):
        ok &= bool(torch.equal(f(*batches[i][:2]), batches[i][2]))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = [f(*batches[i][:2]) for i in range(3, steps + 3)]
    e1.record()
    torch.cuda.synchronize()
    ok &= all(torch.equal(r, batches[i + 3][2]) for i, r in enumerate(out))
    ms = e0.elapsed_time(e1) / steps
    res[mode] = ms
    print(f"{mode}: {ms:.4f} ms/batch  {spec.batch / ms / 1e6:.2f} G ops/s  ok={ok}", flush=True)
    if sh:
        sh.check()
        del sh
    del s, batches, out
    torch.cuda.empty_cache()
print(f"peer-path overhead at world 1: {res['peer'] - res['table']:.4f} ms/batch")
dist.destroy_process_group()
