"""Profiling driver (ncu): one launch each of the config-3 encode variants."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_1805_03709_b200 import BlockHashSet, FaceState, encode_full, encode_keys, face_packs, workloads
dev = torch.device("cuda", 0)
keys_np = workloads.room_block_keys()
keys = torch.from_numpy(keys_np).to(dev)
t = BlockHashSet(1 << 21, 1 << 21, device=dev)
_, pos = t.insert_keys(keys)
pool = torch.empty((t.capacity, 6144), dtype=torch.uint8, device=dev)
for a in range(0, len(keys_np), 1 << 15):
    pool[pos[a:a + (1 << 15)].long()] = workloads.room_tsdf_rows(keys[a:a + (1 << 15)])
st = FaceState(pool)
faces = face_packs(pool, rows=pos)
which = sys.argv[1:] or ["self", "faces", "gather"]
for _ in range(2):
    if "self" in which:
        encode_full(t, pool, keys, state=st)
    if "faces" in which:
        encode_keys(t, pool, keys, faces=faces)
    if "gather" in which:
        encode_keys(t, pool, keys)
torch.cuda.synchronize()
print("done")
