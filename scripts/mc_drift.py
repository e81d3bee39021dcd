"""Config-3 encode: CTA wavefront drift (VSB_MC_DRIFT builds) and an output
digest to compare work-distribution variants (experiments)."""
import ctypes, hashlib, json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_1805_03709_b200 import BlockHashSet, _lib, encode_keys, workloads

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
for _ in range(3):
    mc, q, c = encode_keys(t, pool, keys)
torch.cuda.synchronize()
h = hashlib.sha256(mc.cpu().numpy().tobytes() + q.cpu().numpy().tobytes()).hexdigest()[:16]
times = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    encode_keys(t, pool, keys, mc=mc, q=q)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
out = {"lib": os.environ.get("VSB_LIB", "default"), "digest": h, "ms": round(sorted(times)[2], 3)}
lib = ctypes.CDLL(os.path.abspath(os.environ["VSB_LIB"])) if os.environ.get("VSB_LIB") else None
if lib is not None and hasattr(lib, "vs_mc_drift_read"):
    buf = np.zeros((5, 4096), np.uint64)
    assert lib.vs_mc_drift_read(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    G = int((buf[4] > 0).sum())
    t0 = buf[0][:G][buf[0][:G] > 0].min()
    for m, name in enumerate(["j64", "j256", "j640", "j1024", "end"]):
        v = buf[m][:G].astype(np.int64)
        v = v[v > 0] - int(t0)
        if len(v):
            p = np.percentile(v, [0, 5, 50, 95, 100]) / 1e3
            out[name] = {"n": int(len(v)), "us_p0_p5_p50_p95_p100": [round(float(x), 1) for x in p]}
print(json.dumps(out), flush=True)
