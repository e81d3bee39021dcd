"""Drop-in GPU Marching-Cubes block encoder (mc_encoding.py:34-172 of the
reference), plus the two NEW outputs of the B200 path: the quantised TSDF
bytes and the stream-compacted non-empty cells.

Batched entry points (torch tensors, one launch each):
  encode_blocks(pool, nbr)        dense MC + quantised TSDF + per-block counts
  encode_keys(tsdf_table, pool, keys)  same, neighbour rows from in-kernel
                                  hash lookups (the hash feeds the encoder)
  neighbors(tsdf_table, keys)     the neighbour-row table alone
  compact(mc, counts)             ordered non-empty cells (format A19)
Reference-signature entry points (``recompute_mc_block``,
``recompute_mc_blocks``) gather host TsdfBlocks into a device pool and call
the same kernel.  ``compute_mc_index`` / ``apply_cutoff`` /
``affected_mc_blocks`` are the reference's scalar helpers, kept for API
compatibility (they are not on the measured path).
"""

from __future__ import annotations

import ctypes
from itertools import product
from typing import Callable, Iterable, NamedTuple, Optional

import numpy as np

from . import _lib
from ._lib import check, ptr
from .voxel_model import BLOCK_VOXELS, TSDF_BLOCK_BYTES, block_row

MC_VOXEL_DTYPE = np.dtype([("index", "u1"), ("color", "u1", 3)])
assert MC_VOXEL_DTYPE.itemsize == 4
MC_BLOCK_BYTES = BLOCK_VOXELS * MC_VOXEL_DTYPE.itemsize  # 2048
Q_BLOCK_BYTES = BLOCK_VOXELS  # int8 quantised TSDF per block


class McVoxel(NamedTuple):
    index: int
    color: tuple[int, int, int]


class McBlock:
    """8x8x8 MC voxels, x-fastest (mc_encoding.py:47-80)."""

    __slots__ = ("key", "index", "color")

    def __init__(self, key, index: Optional[np.ndarray] = None, color: Optional[np.ndarray] = None) -> None:
        self.key = key
        self.index = np.zeros(BLOCK_VOXELS, dtype=np.uint8) if index is None else index
        self.color = np.zeros((BLOCK_VOXELS, 3), dtype=np.uint8) if color is None else color

    def is_empty(self) -> bool:
        return not self.index.any()

    def to_bytes(self) -> bytes:
        rec = np.zeros(BLOCK_VOXELS, dtype=MC_VOXEL_DTYPE)
        rec["index"] = self.index
        rec["color"] = self.color
        return rec.tobytes()

    @classmethod
    def from_bytes(cls, key, raw: bytes) -> "McBlock":
        if len(raw) != MC_BLOCK_BYTES:
            raise ValueError(f"MC block payload must be {MC_BLOCK_BYTES} bytes")
        rec = np.frombuffer(raw, dtype=MC_VOXEL_DTYPE)
        return cls(key, rec["index"].copy(), rec["color"].copy())


def compute_mc_index(corners: Iterable[tuple[float, float]]) -> int:
    """Scalar cube index (mc_encoding.py:83-98), API helper."""
    corners = list(corners)
    if len(corners) != 8:
        raise ValueError("a cube has exactly 8 corners")
    index = 0
    for k, (tsdf, weight) in enumerate(corners):
        if weight <= 0:
            return 0
        if tsdf < 0:
            index |= 1 << k
    return index


def apply_cutoff(voxel: McVoxel) -> McVoxel:
    """mc_encoding.py:101-105."""
    if voxel.index == 0 or voxel.index == 255:
        return McVoxel(0, (0, 0, 0))
    return voxel


def affected_mc_blocks(updated) -> list[tuple[int, int, int]]:
    """mc_encoding.py:108-115: the block and its 7 negative neighbours."""
    x, y, z = updated
    return [(x + dx, y + dy, z + dz) for dx, dy, dz in product((0, -1), repeat=3)]


# ----------------------------------------------------------- device entry

def _out(torch, n, device, want, shape, dtype):
    """`want`: False (skip), True (allocate) or a caller tensor to write into."""
    if isinstance(want, torch.Tensor):
        if want.shape != (n,) + shape or want.dtype != dtype or want.device != device or not want.is_contiguous():
            raise ValueError(f"output must be a contiguous {dtype}[{n}, ...{shape}] tensor on {device}")
        return want
    return torch.empty((n,) + shape, dtype=dtype, device=device) if want else None


FACE_BYTES = 48  # face bit-pack per pool row (vs_mc_faces)


def _faces_arg(faces, pool):
    torch = _lib.require_cuda()
    if faces is None:
        return None
    if faces.dtype != torch.uint8 or faces.dim() != 2 or faces.shape[1] != FACE_BYTES or \
            faces.shape[0] < pool.shape[0] or faces.device != pool.device or not faces.is_contiguous():
        raise ValueError("faces must be a contiguous uint8[>= P, 48] tensor on the pool's device")
    return faces


def face_packs(pool, rows=None, faces=None):
    """Face bit-packs of pool rows (the encoder's halo side table): computes
    faces[r] for r in `rows` (int32 tensor; all rows when None) into `faces`
    (allocated uint8[P, 48] when None, zero for rows never computed).
    Returns `faces`.  Call it wherever pool rows change."""
    torch = _lib.require_cuda()
    dev = pool.device
    if faces is None:
        faces = torch.zeros((pool.shape[0], FACE_BYTES), dtype=torch.uint8, device=dev)
    _faces_arg(faces, pool)
    r = None if rows is None else rows.to(dev, torch.int32).contiguous()
    n = pool.shape[0] if r is None else r.shape[0]
    check(_lib.load().vs_mc_faces(ptr(pool.contiguous()), ptr(r), n, ptr(faces), _lib.stream_of(dev)), "mc_faces")
    return faces


def encode_blocks(pool, nbr, *, mc: bool = True, q: bool = True, counts: bool = True, faces=None):
    """Dense encode of N blocks given neighbour rows nbr int32[N,8] into the
    wire-layout TSDF pool uint8[P,6144].  Returns (mc uint8[N,2048] | None,
    q int8[N,512] | None, counts int32[N] | None).  `faces`: the pool's face
    bit-packs (face_packs), current for every neighbour row -- same output,
    less halo traffic."""
    torch = _lib.require_cuda()
    if pool.dtype != torch.uint8 or pool.dim() != 2 or pool.shape[1] != TSDF_BLOCK_BYTES:
        raise ValueError("pool must be uint8[P, 6144]")
    dev = pool.device
    nbr = nbr.to(dev, torch.int32).contiguous().reshape(-1, 8)
    pool = pool.contiguous()
    n = nbr.shape[0]
    mc_t = _out(torch, n, dev, mc, (MC_BLOCK_BYTES,), torch.uint8)
    q_t = _out(torch, n, dev, q, (Q_BLOCK_BYTES,), torch.int8)
    c_t = _out(torch, n, dev, counts, (), torch.int32)
    s = _lib.stream_of(dev)
    f = _faces_arg(faces, pool)
    check(_lib.load().vs_mc_encode(ptr(pool), ptr(f), ptr(nbr), n, ptr(mc_t), ptr(q_t), ptr(c_t), s), "mc_encode")
    return mc_t, q_t, c_t


def encode_keys(tsdf_table, pool, keys, *, mc=True, q=True, counts=True, faces=None, out_rows=None,
                cells: bool = False, cell_cap: Optional[int] = None, n_dev=None):
    """Encode MC blocks `keys` (int32[N,3]); neighbour rows are looked up in
    `tsdf_table` (a BlockHashMap whose positions index `pool`) inside the
    kernel.  `faces`: as for encode_blocks.

    mc / q / counts: True (allocate), False (skip) or a tensor to write.
    out_rows (int32[N]): block i's MC and quantised bytes go to row
    out_rows[i] of `mc` / `q` (caller tensors with >= max(out_rows)+1 rows,
    e.g. a server's MC pool indexed by MC map position).
    n_dev (device int64[1]): encode only the first min(N, n_dev) keys (a
    device-produced count; no host sync).
    cells=True: fused compaction of the non-empty cells in the same launch;
    returns (mc, q, counts, (offsets int32[N], flat int16[M], cell int32[M],
    cursor int64[1])) where block i's cells are [offsets[i], offsets[i] +
    counts[i]) -- else (mc, q, counts)."""
    torch = _lib.require_cuda()
    dev = pool.device
    from .concurrent_hash import _as_keys

    k = _as_keys(keys, dev)
    n = k.shape[0]
    rows = None
    if out_rows is not None:
        rows = out_rows.to(dev, torch.int32).contiguous()
        if rows.shape != (n,):
            raise ValueError("out_rows must be int32[N]")
        if not (isinstance(mc, torch.Tensor) or mc is False) or not (isinstance(q, torch.Tensor) or q is False):
            raise ValueError("out_rows needs caller mc / q tensors (or False)")
        mc_t = mc if isinstance(mc, torch.Tensor) else None
        q_t = q if isinstance(q, torch.Tensor) else None
        for t_, w in ((mc_t, MC_BLOCK_BYTES), (q_t, Q_BLOCK_BYTES)):
            if t_ is not None and (t_.dim() != 2 or t_.shape[1] != w or not t_.is_contiguous() or t_.device != dev):
                raise ValueError("mc / q pools must be contiguous [P, 2048] uint8 / [P, 512] int8 on the pool's device")
    else:
        mc_t = _out(torch, n, dev, mc, (MC_BLOCK_BYTES,), torch.uint8)
        q_t = _out(torch, n, dev, q, (Q_BLOCK_BYTES,), torch.int8)
    c_t = _out(torch, n, dev, counts if isinstance(counts, torch.Tensor) else (bool(counts) or cells), (), torch.int32)
    cur = offs = flat = cm = None
    cap = 0
    if cells:
        cap = int(cell_cap) if cell_cap is not None else n * 512
        cur = torch.zeros(1, dtype=torch.int64, device=dev)
        offs = torch.empty(n, dtype=torch.int32, device=dev)
        flat = torch.empty(max(cap, 1), dtype=torch.int16, device=dev)
        cm = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    s = tsdf_table._stream()
    f = _faces_arg(faces, pool)
    check(_lib.load().vs_mc_encode_keys_ex(tsdf_table.handle, ptr(pool), ptr(f), ptr(k), n, ptr(n_dev), ptr(rows),
                                           ptr(mc_t),
                                           ptr(q_t), ptr(c_t), ptr(cur), ptr(offs), ptr(flat), ptr(cm), cap,
                                           ctypes.c_void_p(s.cuda_stream)), "mc_encode_keys")
    tsdf_table._done(s)
    if cells:
        return mc_t, q_t, c_t, (offs, flat, cm, cur)
    return mc_t, q_t, c_t


def neighbors(tsdf_table, keys):
    """nbr int32[N,8]: position of key + (c&1, c>>1&1, c>>2&1) or -1."""
    torch = _lib.require_cuda()
    from .concurrent_hash import _as_keys

    k = _as_keys(keys, tsdf_table.device)
    out = torch.empty((k.shape[0], 8), dtype=torch.int32, device=k.device)
    s = tsdf_table._stream()
    check(_lib.load().vs_mc_neighbors(tsdf_table.handle, ptr(k), k.shape[0], ptr(out),
                                      ctypes.c_void_p(s.cuda_stream)), "mc_neighbors")
    tsdf_table._done(s)
    return out


def compact(mc, counts, cell_cap: Optional[int] = None):
    """Non-empty cells (format A19): (offsets int64[N+1], flat int16[M]
    (uint16 bit pattern), cells int32[M] = {index, r, g, b} little-endian)."""
    torch = _lib.require_cuda()
    dev = mc.device
    n = mc.shape[0]
    lib = _lib.load()
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    work = torch.empty(max(1, lib.vs_scan_workspace_bytes(n) // 8), dtype=torch.int64, device=dev)
    s = _lib.stream_of(dev)
    counts = counts.to(torch.int32).contiguous()
    check(lib.vs_mc_compact(ptr(mc), ptr(counts), n, ptr(offsets), None, None, 0, ptr(work), s), "mc_compact")
    total = int(offsets[n].item()) if cell_cap is None else cell_cap
    flat = torch.empty(max(total, 1), dtype=torch.int16, device=dev)
    cells = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    check(lib.vs_mc_compact(ptr(mc), ptr(counts), n, ptr(offsets), ptr(flat), ptr(cells), total, ptr(work), s),
          "mc_compact")
    return offsets, flat[:total], cells[:total]


def pack_mc_batch(keys, pos, mc_pool):
    """MC_BATCH payload (wire.py:292-299) straight from the device MC pool:
    u32 count + per block <3i key + 2,048 MC bytes at mc_pool[pos].
    Returns a device uint8 tensor of 4 + 2060*n bytes."""
    torch = _lib.require_cuda()
    dev = mc_pool.device
    from .concurrent_hash import _as_keys

    k = _as_keys(keys, dev)
    p = pos.to(dev, torch.int32).contiguous()
    n = k.shape[0]
    out = torch.empty(4 + (MC_BLOCK_BYTES + 12) * n, dtype=torch.uint8, device=dev)
    check(_lib.load().vs_mc_pack(ptr(k), ptr(p), n, ptr(mc_pool), ptr(out), _lib.stream_of(dev)), "mc_pack")
    return out


def _pool_from_blocks(torch, blocks, device):
    rows = np.stack([block_row(b) for b in blocks]) if blocks else np.zeros((1, TSDF_BLOCK_BYTES), np.uint8)
    return torch.from_numpy(rows).to(device)


def recompute_mc_blocks(keys, tsdf_lookup: Callable, device=None) -> list[McBlock]:
    """Batched ``recompute_mc_block`` over host lookups: every distinct TSDF
    block the keys touch is copied once into a device pool, then ONE encode
    launch computes all blocks."""
    torch = _lib.require_cuda()
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    keys = [tuple(k) for k in keys]
    rows: dict = {}
    blocks = []
    nbr = np.full((len(keys), 8), -1, dtype=np.int32)
    for i, (x, y, z) in enumerate(keys):
        for c in range(8):
            nk = (x + (c & 1), y + ((c >> 1) & 1), z + ((c >> 2) & 1))
            r = rows.get(nk)
            if r is None:
                blk = tsdf_lookup(nk)
                if blk is None:
                    rows[nk] = -1
                    continue
                r = rows[nk] = len(blocks)
                blocks.append(blk)
            nbr[i, c] = r
    if not keys:
        return []
    pool = _pool_from_blocks(torch, blocks, device)
    mc, _, _ = encode_blocks(pool, torch.from_numpy(nbr).to(device), q=False, counts=False)
    rec = mc.cpu().numpy().view(MC_VOXEL_DTYPE).reshape(len(keys), BLOCK_VOXELS)
    return [McBlock(k, rec[i]["index"].copy(), rec[i]["color"].copy()) for i, k in enumerate(keys)]


def recompute_mc_block(key, tsdf_lookup: Callable) -> McBlock:
    """Full 512-voxel recompute of one MC block (mc_encoding.py:145-172)."""
    return recompute_mc_blocks([key], tsdf_lookup)[0]
