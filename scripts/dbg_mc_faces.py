"""Debug/parity check of the face-pack encoder at a size where every CTA
crosses lookup batches: room-corner blocks, packs vs scattered halo."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1805_03709_b200 import BlockHashSet, encode_keys, encode_blocks, face_packs, neighbors, workloads
dev = torch.device("cuda", 0)
nmax = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
keys = workloads.room_block_keys()[:nmax]
kt = torch.from_numpy(keys).to(dev)
rows = workloads.room_tsdf_rows(kt)
tt = BlockHashSet(1 << 18, 1 << 18); _, pos = tt.insert_keys(keys)
pool = torch.zeros((tt.capacity, 6144), dtype=torch.uint8, device=dev); pool[pos.long()] = rows
fp = face_packs(pool, rows=pos)
torch.cuda.synchronize(); print("packs ok", flush=True)
mc, q, c = encode_keys(tt, pool, keys)
torch.cuda.synchronize(); print("plain ok", flush=True)
if os.environ.get("SKIP_NBR") != "1":
    nb = neighbors(tt, keys)
    mc4, q4, c4 = encode_blocks(pool, nb, faces=fp)
    torch.cuda.synchronize(); print("nbr+faces", torch.equal(mc, mc4), torch.equal(q, q4), torch.equal(c, c4), flush=True)
mc3, q3, c3 = encode_keys(tt, pool, keys, faces=fp)
torch.cuda.synchronize(); print("keys+faces", torch.equal(mc, mc3), torch.equal(q, q3), torch.equal(c, c3), flush=True)
