import os, sys
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.getcwd())
import torch, time
from paper_1805_03709_b200 import BlockHashSet, workloads
from paper_1805_03709_b200.shard import OneGpuShardGroup
world = int(sys.argv[1]); live = int(sys.argv[2]); chunk = int(sys.argv[3])
dev = torch.device("cuda", 0)
spec = workloads.MixSpec(live=live)
tabs = [BlockHashSet(spec.bucket_count, spec.excess, device=dev) for _ in range(world)]
g = OneGpuShardGroup(tabs, max_batch=chunk)
z = lambda n: torch.zeros(n, dtype=torch.uint8, device=dev)
for a in range(0, live, chunk):
    b = min(live, a + chunk)
    t0 = time.time()
    out = g.apply([workloads.id_to_key_torch(torch.arange((r << 40) + a, (r << 40) + b, device=dev)) for r in range(world)], [z(b - a)] * world)
    torch.cuda.synchronize()
    print("chunk", a, "secs %.3f" % (time.time() - t0), "created", [int(o.sum()) for o in out], flush=True)
    try:
        g.check(); print("  no timeout")
    except Exception as e:
        print("  TIMEOUT", e)
print("sizes", [t.approx_size() for t in tabs], "total", sum(t.approx_size() for t in tabs), "want", world * live)
