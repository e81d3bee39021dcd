"""Time the config-3 MC encode alone (experiments; the contract bench is bench.py)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_1805_03709_b200 import BlockHashSet, _lib, encode_keys, encode_blocks, face_packs, neighbors, workloads

dev = torch.device("cuda", 0)
keys_np = workloads.room_block_keys()
N = len(keys_np)
keys = torch.from_numpy(keys_np).to(dev)
t = BlockHashSet(1 << 21, 1 << 21, device=dev)
_, pos = t.insert_keys(keys)
t.check_capacity()
pool = torch.empty((t.capacity, 6144), dtype=torch.uint8, device=dev)
for a in range(0, N, 1 << 15):
    pool[pos[a:a + (1 << 15)].long()] = workloads.room_tsdf_rows(keys[a:a + (1 << 15)])
nbr = neighbors(t, keys)
faces = face_packs(pool, rows=pos)
torch.cuda.synchronize()
f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
f0.record()
face_packs(pool, rows=pos, faces=faces)
f1.record()
torch.cuda.synchronize()
ref = None
out = {"lib": os.environ.get("VSB_LIB", "default"), "face_packs_all_rows_ms": round(f0.elapsed_time(f1), 3)}
for name, fn in [("keys", lambda: encode_keys(t, pool, keys)), ("nbr", lambda: encode_blocks(pool, nbr)),
                 ("keys+faces", lambda: encode_keys(t, pool, keys, faces=faces)),
                 ("nbr+faces", lambda: encode_blocks(pool, nbr, faces=faces))]:
    for _ in range(3):
        mc, q, c = fn()
    if ref is None:
        ref = (mc.clone(), q.clone())
    ok = bool(torch.equal(mc, ref[0]) and torch.equal(q, ref[1]))
    times = []
    for _rep in range(5):  # median of 5 rounds of 10 launches
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 10)
    ms = sorted(times)[2]
    out[name] = {"ms": round(ms, 3), "Mblocks_s": round(N / ms / 1e3, 1), "frac": round(N * 8704 / (ms / 1e3) / 6552.6e9, 3), "same": ok}
print(json.dumps(out), flush=True)
