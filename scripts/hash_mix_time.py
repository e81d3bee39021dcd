"""Per-op-kind cost of k_apply on the config-2 table (experiment): the mixed
batches of bench config 2, and the same batches with one kind of mutation
turned into finds.  Each variant runs on a fresh table.  Prints us per
launch (library profiler)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_1805_03709_b200 import BlockHashSet, _lib, workloads

dev = torch.device("cuda", 0)
spec = workloads.MixSpec()


def run(label, transform, n=6):
    s = BlockHashSet(spec.bucket_count, spec.excess, device=dev)
    for a in range(0, spec.live, 1 << 22):
        s.insert_keys(workloads.id_to_key_torch(torch.arange(a, min(spec.live, a + (1 << 22)), device=dev)))
    gen = torch.Generator(device=dev)
    gen.manual_seed(3)
    lo, hi = 0, spec.live
    bs = []
    for step in range(n):
        ids, ops, expect = workloads.mix_batch_ids(spec, step, lo, hi, gen, dev)
        bs.append((workloads.id_to_key_torch(ids), transform(ops, expect)))
        lo += spec.counts["erase"]
        hi += spec.counts["fresh"]
    for k, o in bs[:2]:
        s.apply(k, o)
    with _lib.Profile() as prof:
        for k, o in bs[2:]:
            s.apply(k, o)
    ms = prof.ms["hash"] / prof.count["hash"]
    print(f"{label:44s} {ms * 1e3:7.1f} us  {spec.batch / ms / 1e6:6.2f} G ops/s", flush=True)
    del s
    torch.cuda.empty_cache()


fresh_mask = lambda o, e: (o == 0) & (e == 1)
run("mix 50/30/20", lambda o, e: o)
run("no erases (erase -> find)", lambda o, e: torch.where(o == 2, torch.ones_like(o), o))
run("no fresh inserts (fresh -> find)", lambda o, e: torch.where(fresh_mask(o, e), torch.ones_like(o), o))
run("neither (finds + present inserts)", lambda o, e: torch.where((o == 2) | fresh_mask(o, e), torch.ones_like(o), o))
run("all finds", lambda o, e: torch.ones_like(o))
