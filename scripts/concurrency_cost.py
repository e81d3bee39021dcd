"""Cost of the per-table call serialisation: find batches
issued from 1 thread on one stream vs 2 and 4 threads on their own streams
against ONE table (each call is ordered after the table's previous launch,
so launches from different streams serialise on the GPU).  Prints finds/s."""
import os
import sys
import threading
import time

sys.path.insert(0, os.getcwd())
import torch

from paper_1805_03709_b200 import BlockHashSet, workloads

dev = torch.device("cuda", 0)
spec = workloads.MixSpec()
s = BlockHashSet(spec.bucket_count, spec.excess, device=dev)
for a in range(0, spec.live, 1 << 22):
    s.insert_keys(workloads.id_to_key_torch(torch.arange(a, min(spec.live, a + (1 << 22)), device=dev)))
torch.cuda.synchronize()
B, CALLS = 1 << 16, 256
keys = [workloads.id_to_key_torch(torch.randint(0, spec.live, (B,), device=dev)) for _ in range(8)]


def worker(n, out):
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        for i in range(n):
            s.find_keys(keys[i % 8])
        st.synchronize()
    out.append(1)


for threads in (1, 2, 4):
    for rep in range(2):
        torch.cuda.synchronize()
        out = []
        ts = [threading.Thread(target=worker, args=(CALLS // threads, out)) for _ in range(threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{threads} thread(s): {CALLS * B / dt / 1e9:.2f} G finds/s ({CALLS} calls of {B} keys, {dt * 1e3:.1f} ms)")
