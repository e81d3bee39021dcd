"""Experiment: MC encode of the config-3 room with the work list in key order
vs Morton (Z-order) block order -- does processing order fix the halo L2
misses?  Times encode_blocks (neighbour table) and encode_keys."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_1805_03709_b200 import BlockHashSet, encode_blocks, encode_keys, neighbors, workloads

dev = torch.device("cuda", 0)
keys_np = workloads.room_block_keys()
N = len(keys_np)


def morton(k):
    v = (k.astype(np.int64) + (1 << 20)).astype(np.uint64)
    out = np.zeros(len(k), np.uint64)
    for bit in range(21):
        for a in range(3):
            out |= ((v[:, a] >> np.uint64(bit)) & np.uint64(1)) << np.uint64(3 * bit + a)
    return out


keys = torch.from_numpy(keys_np).to(dev)
t = BlockHashSet(1 << 21, 1 << 21, device=dev)
_, pos = t.insert_keys(keys)
pool = torch.empty((t.capacity, 6144), dtype=torch.uint8, device=dev)
for a in range(0, N, 1 << 15):
    pool[pos[a:a + (1 << 15)].long()] = workloads.room_tsdf_rows(keys[a:a + (1 << 15)])
order = torch.from_numpy(np.argsort(morton(keys_np), kind="stable")).to(dev)
res = {}
for name, kk in [("key order", keys), ("morton", keys[order])]:
    nbr = neighbors(t, kk)
    for label, fn in [("nbr", lambda: encode_blocks(pool, nbr)), ("keys", lambda: encode_keys(t, pool, kk))]:
        for _ in range(3):
            fn()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 5)
        ms = sorted(ts)[2]
        res[f"{name}/{label}"] = {"ms": round(ms, 3), "frac": round(N * 8704 / (ms / 1e3) / 6552.6e9, 3)}
    print(json.dumps(res), flush=True)
# parity of the permuted encode
mc0, q0, _ = encode_blocks(pool, neighbors(t, keys))
mc1, q1, _ = encode_blocks(pool, neighbors(t, keys[order]))
print("same bytes under permutation:", bool(torch.equal(mc0[order], mc1) and torch.equal(q0[order], q1)))
