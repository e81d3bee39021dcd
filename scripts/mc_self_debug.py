"""Debug: per-neighbour pack misses of the self-packing full encode (room)."""
import ctypes, os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_1805_03709_b200 import BlockHashSet, FaceState, _lib, encode_full, workloads
dev = torch.device("cuda", 0)
keys_np = workloads.room_block_keys()
keys = torch.from_numpy(keys_np).to(dev)
t = BlockHashSet(1 << 21, 1 << 21, device=dev)
_, pos = t.insert_keys(keys)
pool = torch.empty((t.capacity, 6144), dtype=torch.uint8, device=dev)
for a in range(0, len(keys_np), 1 << 15):
    pool[pos[a:a + (1 << 15)].long()] = workloads.room_tsdf_rows(keys[a:a + (1 << 15)])
st = FaceState(pool)
lib = _lib.load()
lib.vs_mc_self_debug.restype = ctypes.c_int
lib.vs_mc_self_debug.argtypes = [ctypes.c_void_p]
out = (ctypes.c_uint64 * 8)()
for i in range(3):
    lib.vs_mc_self_debug(out); before = list(out)
    encode_full(t, pool, keys, state=st)
    torch.cuda.synchronize()
    lib.vs_mc_self_debug(out)
    print("launch", i, "misses per c=1..7:", [out[k] - before[k] for k in range(7)])
nb = __import__("paper_1805_03709_b200").neighbors(t, keys)
print("present neighbours per c:", [(nb[:, c] >= 0).sum().item() for c in range(1, 8)])
