"""Two ranks sharing one B200: the sharded hash set with the real GPU tables,
through both exchanges -- "peer" (csrc/shard.cu: the kernels store records
and results straight into CUDA-IPC-mapped windows of the other rank) and
"collective" (all-to-all over the process group; gloo here, staged through
host memory, because NCCL needs one GPU per rank).  Per-op results must
equal the analytic expectation of the A18 workload, every key must live on
its owner, the global size must add up, and duplicate fresh inserts across
ranks must resolve like a sequential replay of rank 0's batch, then rank
1's (the lowest routed index creates)."""

from __future__ import annotations

import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parent.parent

WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"])
import numpy as np, torch, torch.distributed as dist
from paper_1805_03709_b200 import BlockHashSet, workloads
from paper_1805_03709_b200.shard import ShardedBlockHashSet, owner_of

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
exch = os.environ["EXCH"]
dev = torch.device("cuda", 0)
spec = workloads.MixSpec(live=50_000, load_factor=0.7, batch=1 << 14)
shard = ShardedBlockHashSet(BlockHashSet(spec.bucket_count, spec.excess, device=dev), exchange=exch,
                            max_batch=1 << 16)
assert shard.exchange == exch
base = rank << 40
init = workloads.id_to_key_torch(torch.arange(base, base + spec.live, device=dev))
r = shard.apply(init, torch.zeros(spec.live, dtype=torch.uint8, device=dev))
assert int(r.sum()) == spec.live
mine, _ = shard.local.snapshot_tensor()
assert bool((owner_of(mine, world) == rank).all())
gen = torch.Generator(device=dev); gen.manual_seed(rank)
lo, hi = base, base + spec.live
for step in range(4):
    ids, ops, expect = workloads.mix_batch_ids(spec, step, lo, hi, gen, dev)
    ids = torch.where(ids >= workloads.MISS_BASE, ids + (rank << 50), ids)
    res = shard.apply(workloads.id_to_key_torch(ids), ops)
    assert torch.equal(res, expect), (rank, step, int((res != expect).sum()))
    lo += spec.counts["erase"]; hi += spec.counts["fresh"]
assert shard.size() == world * spec.live

# duplicate fresh inserts across and within ranks: the same 300 new keys on
# both ranks, each twice on a rank (positions i and i + 300); finds of them
# in the same batch would break A18, so only inserts
shared = workloads.id_to_key_torch(torch.arange(7 << 45, (7 << 45) + 300, device=dev))
keys = torch.cat([shared, shared])
r = shard.apply(keys, torch.zeros(600, dtype=torch.uint8, device=dev))
want = torch.zeros(600, dtype=torch.uint8, device=dev)
if rank == 0:
    want[:300] = 1
assert torch.equal(r, want), (rank, r.sum().item())
# empty batch on one rank, a batch on the other: still collective-safe
if rank == 0:
    r = shard.apply(shared[:0], torch.zeros(0, dtype=torch.uint8, device=dev))
    assert r.numel() == 0
else:
    r = shard.apply(shared, torch.full((300,), 2, dtype=torch.uint8, device=dev))
    assert int(r.sum()) == 300
assert shard.size() == world * spec.live
shard.check()
a = shard.local.audit()
assert a["duplicates"] == 0 and a["unreachable_live"] == 0
print("RANK_OK", rank, flush=True)
dist.destroy_process_group()
'''


@pytest.mark.parametrize("exch,port", [("peer", 29546), ("collective", 29544)])
def test_two_ranks_one_gpu_routing(tmp_path, dev, exch, port):
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, ROOT=str(ROOT), OMP_NUM_THREADS="1", EXCH=exch)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(w)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert out.count("RANK_OK") == 2, out[-3000:]


def test_peer_single_rank_equals_table(tmp_path, dev):
    """world 1: the peer path (partition, self-window, routed apply, return)
    gives exactly the plain table's per-op results on the config-2 mix."""
    import torch
    import torch.distributed as dist

    from paper_1805_03709_b200 import BlockHashSet, workloads
    from paper_1805_03709_b200.shard import ShardedBlockHashSet

    if not dist.is_initialized():
        dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    try:
        spec = workloads.MixSpec(live=200_000, load_factor=0.7, batch=1 << 16)
        a = BlockHashSet(spec.bucket_count, spec.excess, device=dev)
        b = BlockHashSet(spec.bucket_count, spec.excess, device=dev)
        sh = ShardedBlockHashSet(b, exchange="peer", max_batch=spec.live)
        init = workloads.id_to_key_torch(torch.arange(spec.live, device=dev))
        a.insert_keys(init)
        assert int(sh.apply(init, torch.zeros(spec.live, dtype=torch.uint8, device=dev)).sum()) == spec.live
        gen = torch.Generator(device=dev)
        gen.manual_seed(5)
        lo, hi = 0, spec.live
        for step in range(3):
            ids, ops, expect = workloads.mix_batch_ids(spec, step, lo, hi, gen, dev)
            k = workloads.id_to_key_torch(ids)
            ra = a.apply(k, ops)[0]
            rb = sh.apply(k, ops)
            assert torch.equal(ra, expect) and torch.equal(rb, expect)
            lo += spec.counts["erase"]
            hi += spec.counts["fresh"]
        # duplicates inside one batch: lowest index creates, as the table
        k = workloads.id_to_key_torch(torch.arange(1 << 44, (1 << 44) + 1000, device=dev))
        k = torch.cat([k, k.flip(0), k])
        z = torch.zeros(k.shape[0], dtype=torch.uint8, device=dev)
        assert torch.equal(a.apply(k, z)[0], sh.apply(k, z))
        ka, _ = a.snapshot_tensor()
        kb, _ = b.snapshot_tensor()
        assert a.approx_size() == b.approx_size()
        assert set(map(tuple, ka.tolist())) == set(map(tuple, kb.tolist()))
        sh.check()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,big", [(3, False), (8, False), (3, True), (8, True)])
def test_peer_route_world_on_one_gpu(dev, world, big):
    """An 8-rank (and a 3-rank) node simulated in one process on one GPU:
    every rank's batch on its own stream through the real windows, flags and
    kernels (OneGpuShardGroup).  Per-op results equal the A18 expectation,
    every key lives on its owner, sizes add up, cross-rank duplicate fresh
    inserts resolve to the lowest rank, and every table audits clean.
    big: 1 GiB tables, so the route partitions by (owner, bucket region) and
    owners apply region by region (shard.cu VSB_SHARD_REGIONS)."""
    import torch

    from paper_1805_03709_b200 import BlockHashSet, workloads
    from paper_1805_03709_b200.shard import OneGpuShardGroup, owner_of

    spec = workloads.MixSpec(live=40_000, load_factor=0.7, batch=1 << 13)
    nb, ex = (1 << 25, 1 << 25) if big else (spec.bucket_count, spec.excess)
    tabs = [BlockHashSet(nb, ex, device=dev) for _ in range(world)]
    g = OneGpuShardGroup(tabs, max_batch=spec.live)
    z = lambda n: torch.zeros(n, dtype=torch.uint8, device=dev)  # noqa: E731
    init = [workloads.id_to_key_torch(torch.arange(r << 40, (r << 40) + spec.live, device=dev)) for r in range(world)]
    res = g.apply(init, [z(spec.live)] * world)
    torch.cuda.synchronize()
    assert all(int(x.sum()) == spec.live for x in res)
    for r, t in enumerate(tabs):
        mine, _ = t.snapshot_tensor()
        assert bool((owner_of(mine, world) == r).all()), r
    gens = [torch.Generator(device=dev) for _ in range(world)]
    for r, gg in enumerate(gens):
        gg.manual_seed(100 + r)
    lo = [r << 40 for r in range(world)]
    hi = [(r << 40) + spec.live for r in range(world)]
    for step in range(3):
        ks, os_, ex = [], [], []
        for r in range(world):
            ids, ops, expect = workloads.mix_batch_ids(spec, step, lo[r], hi[r], gens[r], dev)
            ids = torch.where(ids >= workloads.MISS_BASE, ids + (r << 50), ids)
            ks.append(workloads.id_to_key_torch(ids))
            os_.append(ops)
            ex.append(expect)
            lo[r] += spec.counts["erase"]
            hi[r] += spec.counts["fresh"]
        out = g.apply(ks, os_)
        torch.cuda.synchronize()
        for r in range(world):
            assert torch.equal(out[r], ex[r]), (world, step, r, int((out[r] != ex[r]).sum()))
    assert sum(t.approx_size() for t in tabs) == world * spec.live
    # the same 500 new keys on every rank (twice each): rank 0's first copy creates
    shared = workloads.id_to_key_torch(torch.arange(9 << 45, (9 << 45) + 500, device=dev))
    both = torch.cat([shared, shared])
    out = g.apply([both] * world, [z(1000)] * world)
    torch.cuda.synchronize()
    want0 = torch.cat([torch.ones(500, dtype=torch.uint8, device=dev), z(500)])
    assert torch.equal(out[0], want0)
    for r in range(1, world):
        assert int(out[r].sum()) == 0
    # ragged: empty batch on some ranks
    ks = [shared[: (r % 3) * 100] for r in range(world)]
    out = g.apply(ks, [torch.ones(k.shape[0], dtype=torch.uint8, device=dev) for k in ks])
    torch.cuda.synchronize()
    for r in range(world):
        assert int(out[r].sum()) == ks[r].shape[0]
    g.check()
    for t in tabs:
        a = t.audit()
        assert a["duplicates"] == 0 and a["unreachable_live"] == 0


def test_peer_route_timeout_is_loud(dev):
    """A collective call only one rank makes: that rank's device-side wait
    gives up after the (shortened) timeout instead of hanging the GPU, and
    check() raises."""
    import ctypes

    import torch

    from paper_1805_03709_b200 import BlockHashSet, _lib, workloads
    from paper_1805_03709_b200.shard import OneGpuShardGroup

    tabs = [BlockHashSet(1 << 12, 1 << 12, device=dev) for _ in range(2)]
    g = OneGpuShardGroup(tabs, max_batch=1024)
    lib = _lib.load()
    for h in g.shards:
        _lib.check(lib.vs_shard_set_timeout_ms(h, 200))
    k = workloads.id_to_key_torch(torch.arange(100, device=dev))
    o = torch.zeros(100, dtype=torch.uint8, device=dev)
    out = torch.empty(100, dtype=torch.uint8, device=dev)
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(lib.vs_shard_apply(g.shards[0], _lib.ptr(k), _lib.ptr(o), 100, _lib.ptr(out), st))  # rank 1 never calls
    torch.cuda.synchronize()
    with pytest.raises(RuntimeError, match="timeout"):
        _lib.check(lib.vs_shard_check(g.shards[0]), "vs_shard")
