"""numpy-facing wrappers of the C oracle + pure-Python stream-set oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from __future__ import annotations

import ctypes
import itertools
from collections import deque
from typing import Iterable, Optional

import numpy as np

from .cbuild import build

_lib = None
_vp = ctypes.c_void_p


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(build()))
        sig = {
            "oh_hash": (ctypes.c_uint32, [ctypes.c_int32] * 3 + [ctypes.c_uint32]),
            "oh_hash_batch": (None, [_vp, ctypes.c_uint64, ctypes.c_uint32, _vp]),
            "oh_create": (_vp, [ctypes.c_uint32, ctypes.c_uint32]),
            "oh_destroy": (None, [_vp]),
            "oh_clear": (None, [_vp]),
            "oh_size": (ctypes.c_uint64, [_vp]),
            "oh_free_count": (ctypes.c_int64, [_vp]),
            "oh_find": (ctypes.c_int64, [_vp] + [ctypes.c_int32] * 3),
            "oh_insert_batch": (ctypes.c_int64, [_vp, _vp, ctypes.c_uint64, _vp, _vp]),
            "oh_find_batch": (None, [_vp, _vp, ctypes.c_uint64, _vp, _vp]),
            "oh_erase_batch": (None, [_vp, _vp, ctypes.c_uint64, _vp, _vp]),
            "oh_apply_batch": (ctypes.c_int64, [_vp, _vp, _vp, ctypes.c_uint64, _vp, _vp]),
            "oh_apply_batch_mt": (ctypes.c_int64, [_vp, _vp, _vp, ctypes.c_uint64, _vp, _vp, ctypes.c_int]),
            "oh_snapshot": (ctypes.c_uint64, [_vp, _vp, _vp, ctypes.c_uint64]),
            "oh_extract": (ctypes.c_uint64, [_vp, ctypes.c_uint64, ctypes.c_uint64, _vp]),
            "oh_occ": (_vp, [_vp]),
            "oh_next": (_vp, [_vp]),
            "oh_stack": (_vp, [_vp]),
            "oh_capacity": (ctypes.c_uint32, [_vp]),
            "om_quantise": (ctypes.c_int8, [ctypes.c_float, ctypes.c_float]),
            "om_encode_block": (None, [_vp, _vp, _vp, _vp, _vp]),
            "om_encode": (None, [_vp, _vp, ctypes.c_uint64, _vp, _vp, _vp, ctypes.c_int]),
            "om_compact": (ctypes.c_uint64, [_vp, ctypes.c_uint64, _vp, _vp, _vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_vp)


def _keys(keys) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(keys, dtype=np.int32).reshape(-1, 3))
    return a


# ------------------------------------------------------------------ hash

def hash_keys(keys, bucket_count: int) -> np.ndarray:
    k = _keys(keys)
    out = np.empty(len(k), dtype=np.uint32)
    lib().oh_hash_batch(_p(k), len(k), bucket_count, _p(out))
    return out


class OracleHashSet:
    """Sequential restatement of concurrent_hash._HashCore (positions exact)."""

    def __init__(self, bucket_count: int, excess_capacity: int) -> None:
        if bucket_count < 1 or excess_capacity < 1:
            raise ValueError("bucket_count and excess_capacity must be >= 1")
        self.bucket_count = bucket_count
        self.excess_capacity = excess_capacity
        self.capacity = bucket_count + excess_capacity
        self._h = lib().oh_create(bucket_count, excess_capacity)
        if not self._h:
            raise MemoryError("oracle table allocation failed")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().oh_destroy(self._h)
            self._h = None

    def insert_batch(self, keys):
        """-> (created u8[N], index i32[N], first_failure or -1)."""
        k = _keys(keys)
        created = np.zeros(len(k), dtype=np.uint8)
        index = np.full(len(k), -1, dtype=np.int32)
        fail = lib().oh_insert_batch(self._h, _p(k), len(k), _p(created), _p(index))
        return created, index, int(fail)

    def find_batch(self, keys):
        k = _keys(keys)
        found = np.zeros(len(k), dtype=np.uint8)
        index = np.zeros(len(k), dtype=np.int32)
        lib().oh_find_batch(self._h, _p(k), len(k), _p(found), _p(index))
        return found, index

    def erase_batch(self, keys):
        k = _keys(keys)
        erased = np.zeros(len(k), dtype=np.uint8)
        index = np.zeros(len(k), dtype=np.int32)
        lib().oh_erase_batch(self._h, _p(k), len(k), _p(erased), _p(index))
        return erased, index

    def apply_batch(self, keys, ops, threads: int = 0):
        """Mixed batch; threads>0 uses the bucket-partitioned parallel mode."""
        k = _keys(keys)
        o = np.ascontiguousarray(np.asarray(ops, dtype=np.uint8))
        result = np.zeros(len(k), dtype=np.uint8)
        index = np.zeros(len(k), dtype=np.int32)
        if threads > 0:
            fail = lib().oh_apply_batch_mt(self._h, _p(k), _p(o), len(k), _p(result), _p(index), threads)
        else:
            fail = lib().oh_apply_batch(self._h, _p(k), _p(o), len(k), _p(result), _p(index))
        return result, index, int(fail)

    def insert_batch_mt(self, keys, threads: int):
        k = _keys(keys)
        result = np.zeros(len(k), dtype=np.uint8)
        index = np.zeros(len(k), dtype=np.int32)
        fail = lib().oh_apply_batch_mt(self._h, _p(k), None, len(k), _p(result), _p(index), threads)
        return result, index, int(fail)

    def snapshot(self):
        """-> (keys i32[M,3], positions i32[M]) in ascending position order."""
        n = int(lib().oh_size(self._h))
        keys = np.zeros((max(n, 1), 3), dtype=np.int32)
        pos = np.zeros(max(n, 1), dtype=np.int32)
        m = lib().oh_snapshot(self._h, _p(keys), _p(pos), n)
        return keys[:m], pos[:m]

    def extract(self, max_n: int, start: int) -> np.ndarray:
        """_extract (concurrent_hash.py:382-402) with the rotation start given."""
        out = np.zeros((max(max_n, 1), 3), dtype=np.int32)
        m = lib().oh_extract(self._h, max_n, start, _p(out))
        return out[:m]

    def size(self) -> int:
        return int(lib().oh_size(self._h))

    def free_count(self) -> int:
        return int(lib().oh_free_count(self._h))

    def clear(self) -> None:
        lib().oh_clear(self._h)

    # white-box views (oracle self-tests only)
    def raw(self):
        cap = self.capacity
        occ = np.ctypeslib.as_array(ctypes.cast(lib().oh_occ(self._h), ctypes.POINTER(ctypes.c_uint8)), (cap,))
        nxt = np.ctypeslib.as_array(ctypes.cast(lib().oh_next(self._h), ctypes.POINTER(ctypes.c_uint32)), (cap,))
        return occ.copy(), nxt.copy()


# ------------------------------------------------------------- MC encode

TSDF_VOXEL = np.dtype([("tsdf", "<f4"), ("weight", "<f4"), ("color", "u1", 3), ("pad", "u1")])
assert TSDF_VOXEL.itemsize == 12


def make_pool(tsdf: np.ndarray, weight: np.ndarray, color: np.ndarray) -> np.ndarray:
    """SoA blocks [P,512] (+ colour [P,512,3]) -> wire-layout pool u8[P,6144]."""
    P = tsdf.shape[0]
    rec = np.zeros((P, 512), dtype=TSDF_VOXEL)
    rec["tsdf"] = tsdf
    rec["weight"] = weight
    rec["color"] = color
    return np.ascontiguousarray(rec.view(np.uint8).reshape(P, 6144))


def neighbor_table(mc_keys, tsdf_keys) -> np.ndarray:
    """nbr[i, c] = row of TSDF key mc_keys[i] + (c&1, c>>1&1, c>>2&1) or -1."""
    index = {tuple(k): r for r, k in enumerate(np.asarray(tsdf_keys).tolist())}
    mk = np.asarray(mc_keys).reshape(-1, 3).tolist()
    out = np.full((len(mk), 8), -1, dtype=np.int32)
    for i, (x, y, z) in enumerate(mk):
        for c in range(8):
            out[i, c] = index.get((x + (c & 1), y + ((c >> 1) & 1), z + ((c >> 2) & 1)), -1)
    return out


def mc_encode(pool: np.ndarray, nbr: np.ndarray, threads: int = 1):
    """-> (mc u8[N,2048], q i8[N,512], counts u32[N])."""
    pool = np.ascontiguousarray(pool, dtype=np.uint8)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    n = nbr.shape[0]
    mc = np.zeros((n, 2048), dtype=np.uint8)
    q = np.zeros((n, 512), dtype=np.int8)
    counts = np.zeros(n, dtype=np.uint32)
    lib().om_encode(_p(pool), _p(nbr), n, _p(mc), _p(q), _p(counts), threads)
    return mc, q, counts


def quantise(tsdf, weight) -> np.ndarray:
    """Normative quantised TSDF (A17), vectorised numpy form of om_quantise."""
    t = np.asarray(tsdf, dtype=np.float32)
    w = np.asarray(weight, dtype=np.float32)
    with np.errstate(invalid="ignore", over="ignore"):
        s = t * np.float32(127.0)
        s = np.where(s > 127, np.float32(127), s)
        s = np.where(s < -127, np.float32(-127), s)
        q = np.rint(np.nan_to_num(s, nan=0.0)).astype(np.int8)
    return np.where((w > 0) & ~np.isnan(t), q, np.int8(-128)).astype(np.int8)


def mc_compact(mc: np.ndarray):
    mc = np.ascontiguousarray(mc, dtype=np.uint8)
    n = mc.shape[0]
    offsets = np.zeros(n + 1, dtype=np.uint64)
    total = lib().om_compact(_p(mc), n, _p(offsets), None, None)
    flat = np.zeros(max(total, 1), dtype=np.uint16)
    cells = np.zeros(max(total, 1), dtype=np.uint32)
    lib().om_compact(_p(mc), n, _p(offsets), _p(flat), _p(cells))
    return offsets, flat[:total], cells[:total]


def mc_encode_numpy(key, lookup):
    """Vectorised numpy restatement of recompute_mc_block (mc_encoding.py:145-172)
    over SoA blocks: lookup(key) -> (tsdf[512], weight[512], color[512,3]) or None.
    Returns the 2048 McBlock bytes."""
    centre = lookup(tuple(key))
    if centre is None:
        return bytes(2048)
    tsdf = np.zeros((9, 9, 9), dtype=np.float32)
    weight = np.zeros((9, 9, 9), dtype=np.float32)
    x, y, z = key
    for dz, dy, dx in itertools.product((0, 1), repeat=3):
        blk = lookup((x + dx, y + dy, z + dz))
        if blk is None:
            continue
        bt = np.asarray(blk[0], dtype=np.float32).reshape(8, 8, 8)
        bw = np.asarray(blk[1], dtype=np.float32).reshape(8, 8, 8)
        zs = slice(8, 9) if dz else slice(0, 8)
        ys = slice(8, 9) if dy else slice(0, 8)
        xs = slice(8, 9) if dx else slice(0, 8)
        zsrc = slice(0, 1) if dz else slice(0, 8)
        ysrc = slice(0, 1) if dy else slice(0, 8)
        xsrc = slice(0, 1) if dx else slice(0, 8)
        tsdf[zs, ys, xs] = bt[zsrc, ysrc, xsrc]
        weight[zs, ys, xs] = bw[zsrc, ysrc, xsrc]
    inside = tsdf < 0
    observed = weight > 0
    index = np.zeros((8, 8, 8), dtype=np.uint16)
    allobs = np.ones((8, 8, 8), dtype=bool)
    for k in range(8):
        dx, dy, dz = k & 1, (k >> 1) & 1, (k >> 2) & 1
        sub = (slice(dz, dz + 8), slice(dy, dy + 8), slice(dx, dx + 8))
        index |= inside[sub].astype(np.uint16) << k
        allobs &= observed[sub]
    index[~allobs] = 0
    index[index == 255] = 0
    flat = index.reshape(512).astype(np.uint8)
    color = np.where((flat != 0)[:, None], np.asarray(centre[2], dtype=np.uint8), 0).astype(np.uint8)
    rec = np.zeros((512, 4), dtype=np.uint8)
    rec[:, 0] = flat
    rec[:, 1:] = color
    return rec.tobytes()


# ----------------------------------------------------------- stream sets

def affected_mc_blocks(key) -> list[tuple[int, int, int]]:
    """mc_encoding.py:108-115: block + 7 negative neighbours, dx slowest."""
    x, y, z = key
    return [(x + dx, y + dy, z + dz) for dx, dy, dz in itertools.product((0, -1), repeat=3)]


def affected_dedup(updated: Iterable) -> list[tuple[int, int, int]]:
    """server.py:304-307: ordered first-occurrence dedup."""
    out: dict = {}
    for k in updated:
        for nb in affected_mc_blocks(tuple(k)):
            out[nb] = None
    return list(out)


class OracleStreamSet:
    """server.py:49-95 with a Python set in place of BlockHashSet (same
    membership semantics) and the same stale-tolerant generation deque."""

    def __init__(self) -> None:
        self.set: set = set()
        self.order: deque = deque()

    def insert(self, key) -> bool:
        key = tuple(key)
        if key in self.set:
            return False
        self.set.add(key)
        self.order.append(key)
        return True

    def insert_many(self, keys) -> int:
        return sum(self.insert(k) for k in keys)

    def remove(self, key) -> bool:
        key = tuple(key)
        if key in self.set:
            self.set.remove(key)
            return True
        return False

    def size(self) -> int:
        return len(self.set)

    def extract_ordered(self, max_n: int) -> list:
        out = []
        while len(out) < max_n:
            try:
                key = self.order.popleft()
            except IndexError:
                break
            if self.remove(key):
                out.append(key)
        return out
