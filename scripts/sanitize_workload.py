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
# one-call server tick (side-stream fork/join) + fused stream tick + set growth
aff, n_aff = core.on_tsdf_batch(keys[20:60], rows[20:60], sync=False); core.check()
from paper_1805_03709_b200 import stream_tick
stream_tick(sets, torch.from_numpy(keys[:200]).to(dev), 32, seeds=[1, 2, 3])
tiny = StreamSet(4, 4, fifo_capacity=64)
fan_out([tiny], keys[:300], sync=True); assert len(tiny) >= 300 if hasattr(tiny, "__len__") else True
# face packs + both encoder halo paths
from paper_1805_03709_b200 import face_packs
fp = face_packs(pool, rows=pos)
mc3, q3, c3 = encode_keys(tt, pool, keys, faces=fp)
mc4, q4, c4 = encode_blocks(pool, nb, faces=fp)
assert torch.equal(mc, mc3) and torch.equal(mc, mc4)
# ticketed work distribution of the encoder (launches of >= 4 lookup batches per CTA)
rk = workloads.room_block_keys()
rk = rk[(rk[:, 0] <= -120) & (rk[:, 2] <= -120)]
rt = BlockHashSet(1 << 17, 1 << 17); _, rpos = rt.insert_keys(rk)
rpool = torch.zeros((rt.capacity, 6144), dtype=torch.uint8, device=dev)
rpool[rpos.long()] = workloads.room_tsdf_rows(torch.from_numpy(rk).to(dev))
encode_keys(rt, rpool, rk); del rpool
# fan-out bounded by a device count
fan_out(sets, keys[:300], n_dev=torch.tensor([123], dtype=torch.int64, device=dev))
# peer-sharded route at world 1 (partition, push, waits, routed apply/post/return)
import tempfile
import torch.distributed as dist
from paper_1805_03709_b200.shard import ShardedBlockHashSet
dist.init_process_group("gloo", init_method=f"file://{tempfile.mkdtemp()}/pg", rank=0, world_size=1)
sh = ShardedBlockHashSet(BlockHashSet(spec.bucket_count, spec.excess), exchange="peer", max_batch=spec.batch)
sh.apply(workloads.id_to_key_torch(torch.arange(spec.live, device=dev)[:spec.batch]),
         torch.zeros(spec.batch, dtype=torch.uint8, device=dev))
r2 = sh.apply(workloads.id_to_key_torch(ids), ops)
sh.check()
# region-ordered partition (tables >= 1 GiB): 2^26 entries, small batch
big = ShardedBlockHashSet(BlockHashSet(1 << 25, 1 << 25), exchange="peer", max_batch=1 << 12)
big.apply(workloads.id_to_key_torch(torch.arange(1 << 12, device=dev)), torch.zeros(1 << 12, dtype=torch.uint8, device=dev))
big.check(); del big
dist.destroy_process_group()
# RC fusion kernels on a small frame
import types
from paper_1805_03709_b200.voxel_model import GpuVoxelModel
depth, color, Rs, ts, (fx, fy, cx, cy, w, h) = workloads.room_frames(1, 64, 48)
intr = types.SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)
cfg = types.SimpleNamespace(voxel_size=0.005, truncation=0.06, max_weight=128.0, alloc_stride=1)
model = GpuVoxelModel(cfg, bucket_count=1 << 14, excess_capacity=1 << 14, device=dev)
d0, c0 = torch.from_numpy(depth[0]).to(dev), torch.from_numpy(color[0]).to(dev)
model.allocate_blocks_tensor(d0, (Rs[0], ts[0]), intr)
model.integrate_frame_tensor(d0, c0, (Rs[0], ts[0]), intr)
torch.cuda.synchronize()
print("SANITIZE_WORKLOAD_OK", flush=True)
