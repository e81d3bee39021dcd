"""Small workload touching every libvsb200 kernel (run under compute-sanitizer)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from paper_1805_03709_b200 import (BlockHashSet, BlockHashMap, StreamSet, GpuServerCore, compact, encode_blocks,
                                   encode_keys, extract_random_many, fan_out, hash_keys, neighbors,
                                   remove_everywhere, workloads, _lib)
dev = torch.device("cuda", 0)
spec = workloads.MixSpec(live=20000, load_factor=0.7, batch=1 << 12)
s = BlockHashSet(spec.bucket_count, spec.excess)
s.insert_keys(workloads.id_to_key_np(np.arange(spec.live)))
gen = torch.Generator(device=dev); gen.manual_seed(1)
ids, ops, exp = workloads.mix_batch_ids(spec, 0, 0, spec.live, gen, dev)
r, _ = s.apply(workloads.id_to_key_torch(ids), ops)
assert torch.equal(r, exp)
s.find_keys(workloads.id_to_key_np(np.arange(100))); s.erase_keys(workloads.id_to_key_np(np.arange(50, 150)))
s.extract_keys(100); s.extract_keys(70000); s.snapshot_tensor(); s.audit(); hash_keys(np.zeros((5, 3), np.int32), 97)
t = BlockHashSet(4, 16)
try:
    t.insert_many_exact([(i, 0, 0) for i in range(40)])
except Exception:
    pass
m = BlockHashMap(64, 64); m.put((1, 2, 3), "a"); m.get((1, 2, 3)); m.remove((1, 2, 3))
keys = workloads.config1_mc_keys()[:2000]
tsdf, weight, color = workloads.random_field(len(keys))
rows = oracle.make_pool(tsdf, weight, color)
tt = BlockHashSet(1 << 12, 1 << 12); _, pos = tt.insert_keys(keys)
pool = torch.zeros((tt.capacity, 6144), dtype=torch.uint8, device=dev); pool[pos.long()] = torch.from_numpy(rows).to(dev)
mc, q, c = encode_keys(tt, pool, keys)
nb = neighbors(tt, keys)
mc2, q2, c2 = encode_blocks(pool, nb)
assert torch.equal(mc, mc2) and torch.equal(q, q2)
compact(mc, c)
sets = [StreamSet(1 << 10, 1 << 10, fifo_capacity=256) for _ in range(3)]
fan_out(sets, keys[:500]); extract_random_many(sets, 64); remove_everywhere(sets, keys[:50])
sets[0].extract_ordered(100); sets[0].fifo_entries(); sets[1].clear()
core = GpuServerCore(1 << 10, 1 << 10, stream_buckets=1 << 9, stream_excess=1 << 9)
cl = core.attach(b"a" * 16)
core.on_tsdf_batch(keys[:20], rows[:20]); core.on_reset_blocks(keys[:5])
torch.cuda.synchronize()
print("SANITIZE_WORKLOAD_OK", flush=True)
