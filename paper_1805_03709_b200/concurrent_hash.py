"""Drop-in GPU replacement of ``voxelstream.concurrent_hash``.

Same public names, constructor signatures, return values and exceptions as
the reference (concurrent_hash.py:35-491); the storage and every operation
run in libvsb200 (hash.cu / hash_ops.cuh) on the GPU.  Each Python call is
one batched launch; the ``*_keys`` / ``apply`` methods take and return torch
tensors and are the fast path (no host sync), the per-key methods exist for
API compatibility and synchronise.

Map payloads: exactly as the reference's ``_values`` list (concurrent_hash.py
:112) they live in an array indexed by entry position, which is stable while
a key is present (:8-13).  For Python objects that array is a host list; the
GPU server core (server.py in this package) uses device tensors instead.
"""

from __future__ import annotations

import ctypes
import random
import threading
from typing import Any, Callable, Iterable, Optional

import numpy as np

from . import _lib
from ._lib import CapacityExhausted, check, ptr

BlockKey = tuple[int, int, int]

# Spatial hash primes, concurrent_hash.py:38-40 (normative).
HASH_P1 = 73856093
HASH_P2 = 19349669
HASH_P3 = 83492791
_MASK32 = 0xFFFFFFFF

__all__ = [
    "BlockKey", "BlockHashMap", "BlockHashSet", "CapacityExhausted", "FreeListStack",
    "HASH_P1", "HASH_P2", "HASH_P3", "hash_key", "hash_keys",
]


def hash_key(key: BlockKey, bucket_count: int) -> int:
    """Bucket index of one key (concurrent_hash.py:49-59).

    Scalar form of the normative arithmetic (uint32 wrapping products, XOR,
    non-negative modulo) for API compatibility; batches go through
    :func:`hash_keys` on the GPU.
    """
    x, y, z = key
    h = ((x * HASH_P1) & _MASK32) ^ ((y * HASH_P2) & _MASK32) ^ ((z * HASH_P3) & _MASK32)
    return h % bucket_count


def hash_keys(keys, bucket_count: int):
    """Batched hash_key on the GPU: int32[N,3] -> int64[N] bucket indices."""
    torch = _lib.require_cuda()
    k = _as_keys(keys, torch.device("cuda", torch.cuda.current_device()))
    out = torch.empty(k.shape[0], dtype=torch.int32, device=k.device)
    check(_lib.load().vs_hash_keys(ptr(k), k.shape[0], bucket_count, ptr(out),
                                   _lib.stream_of(k.device)), "hash_keys")
    return out.to(torch.int64) & _MASK32


class FreeListStack:
    """LIFO pool of free excess-entry indices (concurrent_hash.py:62-82).

    Kept for API compatibility as a plain container.  The GPU tables do not
    use it: their free-list stack is a device array with warp-aggregated pops
    (hash_ops.cuh pop_free) -- see ``BlockHashSet.free_stack``.
    """

    def __init__(self, indices: Iterable[int] = ()) -> None:
        self._slots: list[int] = list(indices)

    def push(self, index: int) -> None:
        self._slots.append(index)

    def pop(self) -> Optional[int]:
        try:
            return self._slots.pop()
        except IndexError:
            return None

    def __len__(self) -> int:
        return len(self._slots)


class _DeviceFreeStack:
    """``len()`` view of a table's device free-list stack."""

    def __init__(self, core: "_HashCore") -> None:
        self._core = core

    def __len__(self) -> int:
        return self._core.free_count()


def _as_keys(keys, device):
    """Anything key-like -> contiguous int32[N,3] tensor on `device`."""
    import torch

    if isinstance(keys, torch.Tensor):
        t = keys
    else:
        if not isinstance(keys, (list, tuple, np.ndarray)):
            keys = list(keys)
        a = np.asarray(keys, dtype=np.int32).reshape(-1, 3) if len(keys) else np.empty((0, 3), np.int32)
        t = torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype != torch.int32:
        t = t.to(torch.int32)
    t = t.reshape(-1, 3)
    if t.device != device:
        t = t.to(device, non_blocking=True)
    return t.contiguous()


# bumped whenever any table records a launch (_HashCore._done, server._mark_done):
# a caller that recorded it right after its own launches knows, while it is
# unchanged, that no table saw a launch since (stream-ordering fast paths)
LAUNCH_GEN = [0]


class _HashCore:
    """One GPU table (bucket region + excess region), shared by set and map."""

    def __init__(self, bucket_count: int = 1 << 20, excess_capacity: int = 1 << 20, *,
                 store_values: bool = False, lock_stripes: int = 1024, device=None) -> None:
        if bucket_count < 1:
            raise ValueError("bucket_count must be >= 1")
        if excess_capacity < 1:
            raise ValueError("excess_capacity must be >= 1")
        if lock_stripes & (lock_stripes - 1):
            raise ValueError("lock_stripes must be a power of two")
        torch = _lib.require_cuda()
        self._torch = torch
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.bucket_count = bucket_count
        self.excess_capacity = excess_capacity
        self.capacity = bucket_count + excess_capacity
        self._lib = _lib.load()
        handle = ctypes.c_void_p()
        check(self._lib.vs_table_create(bucket_count, excess_capacity, self.device.index,
                                        ctypes.byref(handle)), "BlockHashSet")
        self._h = handle
        self._values: Optional[list[Any]] = [None] * self.capacity if store_values else None
        self._mutex = threading.RLock()
        self._last_stream = None
        self._last_sid = None  # raw handle of _last_stream (cheap comparisons)
        self._n_dev = torch.empty(1, dtype=torch.int64, device=self.device)

    # -- lifetime ----------------------------------------------------------

    def __del__(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.vs_table_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    # -- stream ordering: all launches on one table are serialised --------
    # Launches are stream-ordered per table.  When a call comes from a
    # different stream than the table's last launch, the new stream waits for
    # an event recorded on the old one; on the same stream nothing is needed.

    def _stream(self):
        s = self._torch.cuda.current_stream(self.device)
        if self._last_sid is not None and self._last_sid != s.cuda_stream:
            ev = self._torch.cuda.Event()
            ev.record(self._last_stream)
            s.wait_event(ev)
        return s

    def _done(self, s) -> None:
        self._last_stream = s
        self._last_sid = s.cuda_stream
        LAUNCH_GEN[0] += 1

    def _keys(self, keys):
        return _as_keys(keys, self.device)

    # -- batched tensor API (the fast path) --------------------------------

    def insert_keys(self, keys):
        """Batched insert -> (created uint8[N], index int32[N]); asynchronous.

        created follows sequential replay (lowest input index among in-batch
        duplicates creates).  index is -1 for an op that hit an empty free
        list; such failures also raise on the next :meth:`check_capacity`.
        """
        torch = self._torch
        with self._mutex:
            k = self._keys(keys)
            n = k.shape[0]
            created = torch.empty(n, dtype=torch.uint8, device=self.device)
            index = torch.empty(n, dtype=torch.int32, device=self.device)
            s = self._stream()
            check(self._lib.vs_table_insert(self._h, ptr(k), n, ptr(created), ptr(index),
                                            ctypes.c_void_p(s.cuda_stream)), "insert")
            self._done(s)
            return created, index

    def find_keys(self, keys):
        """Batched retrieval -> (found uint8[N], index int32[N]); asynchronous."""
        torch = self._torch
        with self._mutex:
            k = self._keys(keys)
            n = k.shape[0]
            found = torch.empty(n, dtype=torch.uint8, device=self.device)
            index = torch.empty(n, dtype=torch.int32, device=self.device)
            s = self._stream()
            check(self._lib.vs_table_find(self._h, ptr(k), n, ptr(found), ptr(index),
                                          ctypes.c_void_p(s.cuda_stream)), "find")
            self._done(s)
            return found, index

    def erase_keys(self, keys):
        """Batched remove -> (erased uint8[N], vacated index int32[N])."""
        torch = self._torch
        with self._mutex:
            k = self._keys(keys)
            n = k.shape[0]
            erased = torch.empty(n, dtype=torch.uint8, device=self.device)
            index = torch.empty(n, dtype=torch.int32, device=self.device)
            s = self._stream()
            check(self._lib.vs_table_erase(self._h, ptr(k), n, ptr(erased), ptr(index),
                                           ctypes.c_void_p(s.cuda_stream)), "erase")
            self._done(s)
            return erased, index

    def apply(self, keys, ops):
        """Mixed insert/find/erase batch in ONE launch -> (result, index)."""
        torch = self._torch
        with self._mutex:
            k = self._keys(keys)
            o = ops.to(self.device, torch.uint8).contiguous()
            n = k.shape[0]
            if o.shape[0] != n:
                raise ValueError("ops and keys differ in length")
            result = torch.empty(n, dtype=torch.uint8, device=self.device)
            index = torch.empty(n, dtype=torch.int32, device=self.device)
            s = self._stream()
            check(self._lib.vs_table_apply(self._h, ptr(k), ptr(o), n, ptr(result), ptr(index),
                                           ctypes.c_void_p(s.cuda_stream)), "apply")
            self._done(s)
            return result, index

    def check_capacity(self) -> None:
        """Raise CapacityExhausted if an insert since the last check failed."""
        with self._mutex:
            s = self._stream()
            check(self._lib.vs_table_check(self._h, ctypes.c_void_p(s.cuda_stream)))

    def insert_many_exact(self, keys):
        """Insert with the reference's sequential failure semantics.

        Equivalent to ``for k in keys: insert(k)``: on CapacityExhausted the
        keys before the failing one are present, the failing one and all
        later ones are not, and the exception is raised.  Returns
        (created, index) tensors on success.
        """
        torch = self._torch
        k = self._keys(keys)
        created, index = self.insert_keys(k)
        try:
            self.check_capacity()
            return created, index
        except CapacityExhausted:
            pass
        f = int(torch.nonzero(index < 0)[0, 0])
        later = created.clone()
        later[: f + 1] = 0
        undo = k[later.bool()]
        if undo.shape[0]:
            self.erase_keys(undo)
        c1, i1 = self.insert_keys(k[f:f + 1])
        self.check_capacity()  # raises with keys[:f] applied, like the reference
        c2, i2 = self.insert_many_exact(k[f + 1:]) if f + 1 < k.shape[0] else (
            created[:0], index[:0])
        return torch.cat([created[:f], c1, c2]), torch.cat([index[:f], i1, i2])

    def snapshot_tensor(self):
        """Live keys (int32[M,3]) and positions (int32[M]), ascending position."""
        torch = self._torch
        with self._mutex:
            s = self._stream()
            n = self._size_sync(s)
            keys = torch.empty((max(n, 1), 3), dtype=torch.int32, device=self.device)
            pos = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
            check(self._lib.vs_table_snapshot(self._h, ptr(keys), ptr(pos), n, ptr(self._n_dev),
                                              ctypes.c_void_p(s.cuda_stream)), "snapshot")
            self._done(s)
            return keys[:n], pos[:n]

    def audit(self) -> dict[str, int]:
        """Full-scan invariants (replaces the reference's white-box checks)."""
        with self._mutex:
            s = self._stream()
            out = (ctypes.c_uint64 * 6)()
            check(self._lib.vs_table_audit(self._h, ctypes.byref(out), ctypes.c_void_p(s.cuda_stream)))
            self._done(s)
            names = ["live", "reachable_excess", "free", "duplicates", "unreachable_live",
                     "free_reachable"]
            return dict(zip(names, (int(v) for v in out)))

    # -- per-key compatibility path ----------------------------------------

    _OPS = {"vs_table_insert": 0, "vs_table_find": 1, "vs_table_erase": 2}

    def _one(self, fn_name: str, key: BlockKey) -> tuple[int, int]:
        """One key through vs_table_single (pinned staging inside the
        library, one launch, synchronous) -> (flag, position)."""
        with self._mutex:
            s = self._stream()
            k = (ctypes.c_int32 * 3)(*key)
            res = ctypes.c_uint8(0)
            idx = ctypes.c_int32(-1)
            st = self._lib.vs_table_single(self._h, self._OPS[fn_name], ctypes.byref(k), ctypes.byref(res),
                                           ctypes.byref(idx), ctypes.c_void_p(s.cuda_stream))
            if st == _lib.VS_ERR_CAPACITY:
                return 0, -1
            check(st, fn_name)
            return int(res.value), int(idx.value)

    def _insert_pos(self, key: BlockKey) -> tuple[int, bool]:
        created, pos = self._one("vs_table_insert", key)
        if pos < 0:
            raise CapacityExhausted(f"excess list exhausted ({self.excess_capacity} entries)")
        return pos, bool(created)

    def _find(self, key: BlockKey) -> Optional[int]:
        found, pos = self._one("vs_table_find", key)
        return pos if found else None

    def try_insert_once(self, key: BlockKey) -> Optional[int]:
        """concurrent_hash.py:212-249.  The GPU insert has no lock-race
        failure mode (every attempt loops to completion), so this returns the
        entry position, or None only when the free list is exhausted."""
        created, pos = self._one("vs_table_insert", key)
        return None if pos < 0 else pos

    def remove(self, key: BlockKey) -> bool:
        erased, pos = self._one("vs_table_erase", key)
        if erased and self._values is not None:
            self._values[pos] = None
        return bool(erased)

    def __contains__(self, key: BlockKey) -> bool:
        return self._find(key) is not None

    def remove_many(self, keys) -> int:
        """``sum(remove(k) for k in keys)`` in one launch (a per-key remove is
        one GPU round trip); map values of the removed keys are dropped."""
        keys = list(keys) if not hasattr(keys, "shape") else keys
        if len(keys) == 0:
            return 0
        erased, pos = self.erase_keys(keys)
        e = erased.cpu().tolist()
        if self._values is not None:
            with self._mutex:
                for f, p in zip(e, pos.cpu().tolist()):
                    if f:
                        self._values[p] = None
        return int(sum(e))

    def snapshot_keys(self) -> list[BlockKey]:
        keys, _ = self.snapshot_tensor()
        return [tuple(k) for k in keys.cpu().tolist()]

    def _size_sync(self, s) -> int:
        out = ctypes.c_uint64()
        check(self._lib.vs_table_size(self._h, None, ctypes.byref(out), ctypes.c_void_p(s.cuda_stream)))
        return int(out.value)

    def approx_size(self) -> int:
        with self._mutex:
            return self._size_sync(self._stream())

    def free_count(self) -> int:
        with self._mutex:
            s = self._stream()
            out = ctypes.c_uint64()
            check(self._lib.vs_table_free_count(self._h, ctypes.byref(out), ctypes.c_void_p(s.cuda_stream)))
            return int(out.value)

    @property
    def free_stack(self) -> _DeviceFreeStack:
        return _DeviceFreeStack(self)

    def clear(self) -> None:
        with self._mutex:
            s = self._stream()
            check(self._lib.vs_table_clear(self._h, ctypes.c_void_p(s.cuda_stream)), "clear")
            self._done(s)
            if self._values is not None:
                self._values = [None] * self.capacity


class BlockHashSet(_HashCore):
    """Concurrent hash set of block keys (concurrent_hash.py:348-402)."""

    def __init__(self, bucket_count: int = 1 << 20, excess_capacity: int = 1 << 20, *,
                 lock_stripes: int = 1024, device=None) -> None:
        super().__init__(bucket_count, excess_capacity, store_values=False,
                         lock_stripes=lock_stripes, device=device)

    def insert(self, key: BlockKey) -> bool:
        _, created = self._insert_pos(key)
        return created

    def extract_keys(self, max_n: int, seed: Optional[int] = None):
        """Device extract_batch -> int32[m,3] tensor of removed keys.

        Small requests use the windowed single-launch scan
        (vs_stream_extract_random); large ones the full ordered compaction
        (vs_table_extract).  Both start at a seeded random position and take
        live entries in position order, like concurrent_hash.py:387-399."""
        torch = self._torch
        with self._mutex:
            if seed is None:
                seed = random.getrandbits(64)
            seed &= (1 << 64) - 1
            m = max(0, min(int(max_n), self.capacity))
            if m == 0:
                return torch.empty((0, 3), dtype=torch.int32, device=self.device)
            out = torch.empty((m, 3), dtype=torch.int32, device=self.device)
            s = self._stream()
            if m <= (1 << 16):
                handles = (ctypes.c_void_p * 1)(self._h.value)
                seeds = (ctypes.c_uint64 * 1)(seed)
                check(self._lib.vs_stream_extract_random(handles, 1, m, seeds, ptr(out), ptr(self._n_dev),
                                                         ctypes.c_void_p(s.cuda_stream)), "extract")
            else:
                check(self._lib.vs_table_extract(self._h, m, seed, ptr(out), ptr(self._n_dev),
                                                 ctypes.c_void_p(s.cuda_stream)), "extract")
            self._done(s)
            s.synchronize()
            n = int(self._n_dev.item())
            return out[:n]

    def extract_visible_keys(self, max_n: int, planes, margin: float, block_size: float,
                             seed: Optional[int] = None):
        """extract_matching with the server's frustum-AABB predicate
        (server.py:365-387) evaluated on the device -> int32[m,3] tensor.
        planes: (6,4) float64 (Frustum._planes), margin/block_size: floats."""
        torch = self._torch
        with self._mutex:
            if seed is None:
                seed = random.getrandbits(64)
            m = max(0, min(int(max_n), self.capacity))
            if m == 0:
                return torch.empty((0, 3), dtype=torch.int32, device=self.device)
            pl = np.ascontiguousarray(np.asarray(planes, dtype=np.float64).reshape(24))
            out = torch.empty((m, 3), dtype=torch.int32, device=self.device)
            s = self._stream()
            handles = (ctypes.c_void_p * 1)(self._h.value)
            seeds = (ctypes.c_uint64 * 1)(seed & ((1 << 64) - 1))
            check(self._lib.vs_stream_extract_visible(handles, 1, m, seeds, (ctypes.c_double * 24)(*pl),
                                                      float(margin), float(block_size), ptr(out), ptr(self._n_dev),
                                                      ctypes.c_void_p(s.cuda_stream)), "extract_visible")
            self._done(s)
            s.synchronize()
            return out[: int(self._n_dev.item())]

    def extract_visible(self, max_n: int, planes, margin: float, block_size: float) -> list[BlockKey]:
        if max_n <= 0:
            return []
        return [tuple(k) for k in self.extract_visible_keys(max_n, planes, margin, block_size).cpu().tolist()]

    def extract_batch(self, max_n: int) -> list[BlockKey]:
        """Remove and return up to max_n keys from a rotating random start
        (concurrent_hash.py:366-374, 382-402)."""
        if max_n <= 0:
            return []
        return [tuple(k) for k in self.extract_keys(max_n).cpu().tolist()]

    def extract_matching(self, max_n: int, predicate: Callable[[BlockKey], bool]) -> list[BlockKey]:
        """concurrent_hash.py:376-380 with an arbitrary host predicate.

        A Python callable cannot run on the device, so this is the
        compatibility path: device snapshot -> host predicate in rotated
        position order -> one batched device remove.  The server's frustum
        predicate has a device version (server.py in this package).
        """
        if max_n <= 0:
            return []
        keys, pos = self.snapshot_tensor()
        if keys.shape[0] == 0:
            return []
        start = random.randrange(self.capacity)
        pos_l = pos.cpu().tolist()
        keys_l = [tuple(k) for k in keys.cpu().tolist()]
        import bisect

        split = bisect.bisect_left(pos_l, start)
        order = list(range(split, len(keys_l))) + list(range(split))
        picked = []
        for i in order:
            if len(picked) >= max_n:
                break
            if predicate(keys_l[i]):
                picked.append(keys_l[i])
        if not picked:
            return []
        erased, _ = self.erase_keys(picked)
        ok = erased.cpu().tolist()
        return [k for k, e in zip(picked, ok) if e]


class BlockHashMap(_HashCore):
    """Concurrent hash map from block key to a payload (concurrent_hash.py:405-491)."""

    def __init__(self, bucket_count: int = 1 << 20, excess_capacity: int = 1 << 20, *,
                 lock_stripes: int = 1024, device=None) -> None:
        super().__init__(bucket_count, excess_capacity, store_values=True,
                         lock_stripes=lock_stripes, device=device)

    def insert(self, key: BlockKey, value: Any) -> int:
        """Insert if absent; an existing payload is kept; returns the position."""
        with self._mutex:
            pos, created = self._insert_pos(key)
            if created:
                self._values[pos] = value
            return pos

    def put(self, key: BlockKey, value: Any) -> int:
        """Upsert (concurrent_hash.py:427-447)."""
        with self._mutex:
            pos, _ = self._insert_pos(key)
            self._values[pos] = value
            return pos

    def get(self, key: BlockKey, default: Any = None) -> Any:
        with self._mutex:
            pos = self._find(key)
            return default if pos is None else self._values[pos]

    def get_many(self, keys, default: Any = None) -> list:
        """``[get(k) for k in keys]`` with ONE batched lookup (a per-key get
        is one GPU round trip)."""
        keys = list(keys)
        if not keys:
            return []
        found, pos = self.find_keys(keys)
        with self._mutex:
            return [self._values[p] if f else default for f, p in zip(found.cpu().tolist(), pos.cpu().tolist())]

    def get_or_create(self, key: BlockKey, factory: Callable[[], Any]) -> tuple[Any, bool]:
        """Exactly one caller creates (concurrent_hash.py:462-478)."""
        with self._mutex:
            pos, created = self._insert_pos(key)
            if created:
                self._values[pos] = factory()
            return self._values[pos], created

    def value_at(self, pos: int) -> Any:
        return self._values[pos]

    def snapshot_items(self) -> list[tuple[BlockKey, Any]]:
        keys, pos = self.snapshot_tensor()
        vals = self._values
        return [(tuple(k), vals[p]) for k, p in zip(keys.cpu().tolist(), pos.cpu().tolist())]
