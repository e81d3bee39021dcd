"""Two ranks sharing one B200: the sharded router with the real GPU tables
(exchanges over gloo, staged through host memory -- NCCL needs one GPU per
rank).  Per-op results must equal the analytic expectation of the A18
workload, every key must live on its owner, the global size must add up."""

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
dev = torch.device("cuda", 0)
spec = workloads.MixSpec(live=50_000, load_factor=0.7, batch=1 << 14)
shard = ShardedBlockHashSet(BlockHashSet(spec.bucket_count, spec.excess, device=dev))
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
    assert torch.equal(res, expect), (rank, step)
    lo += spec.counts["erase"]; hi += spec.counts["fresh"]
assert shard.size() == world * spec.live
a = shard.local.audit()
assert a["duplicates"] == 0 and a["unreachable_live"] == 0
print("RANK_OK", rank, flush=True)
dist.destroy_process_group()
'''


def test_two_ranks_one_gpu_routing(tmp_path, dev):
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, ROOT=str(ROOT), OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29544", str(w)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert out.count("RANK_OK") == 2, out[-3000:]
