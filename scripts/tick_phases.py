"""Config-4 tick phase breakdown (VSB_TICK_PROF build of k_stream_tick):
per CTA, the globaltimer at launch start, after the dedup, after the
thread-0 insert, after the FIFO append, after the extraction scan and at the
end.  Prints the median / max over the 64 CTAs of each phase (us)."""
import ctypes, json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_1805_03709_b200 import StreamSet, fan_out, stream_tick, workloads

dev = torch.device("cuda", 0)
scene = workloads.room_block_keys()
keys = torch.from_numpy(scene).to(dev)
C, U, X = 16, 512, 512
clients = [StreamSet(1 << 21, 1 << 21, device=dev, fifo_capacity=1 << 22) for _ in range(C)]
fan_out(clients, keys)
rng = np.random.default_rng(0)
lib = ctypes.CDLL(os.path.abspath(os.environ["VSB_LIB"]))
rows = []
times = []
for t in range(60):
    upd = torch.from_numpy(scene[rng.integers(0, len(scene), U)]).to(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    stream_tick(clients, upd, X, seeds=[t * C + c for c in range(C)])
    e1.record()
    torch.cuda.synchronize()
    if t < 10:
        continue
    times.append(e0.elapsed_time(e1) * 1e3)
    buf = np.zeros((8, 256), np.uint64)
    assert lib.vs_tick_prof_read(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    b = buf[:8, :4 * C].astype(np.int64)
    t0 = b[0].min()
    rows.append(np.stack([b[0] - t0, b[1] - b[0], b[2] - b[1], b[3] - b[2], b[4] - b[3], b[5] - b[4], b[5] - t0,
                          b[6] - b[0], b[7] - b[6], b[1] - b[7]]))
r = np.stack(rows) / 1e3  # ticks x 7 x CTAs, us
names = ["start skew", "dedup", "insert (thread 0)", "scan+append", "extract scan", "removals", "end (from first start)",
         "dedup: load+stage", "dedup: hash probes", "dedup: flags+scan+compact"]
out = {"event_us_median": round(float(np.median(times)), 1)}
for i, nm in enumerate(names):
    out[nm] = {"median": round(float(np.median(r[:, i])), 2), "p90": round(float(np.percentile(r[:, i], 90)), 2),
               "max": round(float(r[:, i].max()), 2)}
print(json.dumps(out), flush=True)
