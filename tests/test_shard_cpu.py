"""Multi-process (gloo, world size 2) test of the key-hash sharding router
(paper_1805_03709_b200/shard.py).  The local per-rank table is a test-side
stand-in backed by the C oracle (no GPU here); the routing, the all-to-all
exchanges and the scatter back are the product code.
"""

from __future__ import annotations

import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent

WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"])
import numpy as np, torch, torch.distributed as dist
import oracle
from paper_1805_03709_b200 import workloads
from paper_1805_03709_b200.shard import ShardedBlockHashSet, owner_of

class OracleTable:  # test stand-in for the rank's GPU table
    def __init__(self, n, excess):
        self.t = oracle.OracleHashSet(n, excess)
    def apply(self, keys, ops):
        r, idx, fail = self.t.apply_batch(keys.numpy(), ops.numpy())
        assert fail == -1
        return torch.from_numpy(r), torch.from_numpy(idx)
    def approx_size(self):
        return self.t.size()

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
spec = workloads.MixSpec(live=20_000, load_factor=0.7, batch=1 << 12)
shard = ShardedBlockHashSet(OracleTable(spec.bucket_count, spec.excess))
base = rank << 40
init = workloads.id_to_key_np(np.arange(base, base + spec.live))
r = shard.apply(torch.from_numpy(init), torch.zeros(spec.live, dtype=torch.uint8))
assert int(r.sum()) == spec.live
# every rank's keys landed on their owners only
mine = shard.local.t.snapshot()[0]
assert bool((owner_of(torch.from_numpy(mine), world) == rank).all())
rng = np.random.default_rng(rank)
lo, hi = base, base + spec.live
for step in range(3):
    ids, ops, expect = workloads.mix_batch_ids_np(spec, step, lo, hi, rng)
    ids = np.where(ids >= workloads.MISS_BASE, ids + (rank << 50), ids)
    keys = workloads.id_to_key_np(ids)
    res = shard.apply(torch.from_numpy(keys), torch.from_numpy(ops))
    assert np.array_equal(res.numpy(), expect), (rank, step)
    lo += spec.counts["erase"]; hi += spec.counts["fresh"]
total = shard.size()
assert total == world * spec.live, total
print("RANK_OK", rank, total, flush=True)
dist.destroy_process_group()
'''


def test_two_rank_gloo_routing(tmp_path):
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, ROOT=str(ROOT), OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", str(w)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert out.count("RANK_OK") == 2, out[-3000:]
