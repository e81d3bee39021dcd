"""GPU stream sets and the server's data-parallel update path.

Mirrors the hot half of the reference server (server.py):
  StreamSet        :49-95    device hash set + device generation-order FIFO
  fan_out          :314-315  insert_many of the recomputed keys into EVERY
                             client set in one launch (set difference +
                             ordered FIFO append per client)
  GpuServerCore    :221-249, 299-315, 425-436
                   on_tsdf_batch (TSDF put -> affected dedup -> MC recompute
                   -> MC put -> fan-out), fresh/returning attach, resets.
The control plane (sockets, negotiation, pose/texture relays, stats) stays
in the reference and is out of scope.
"""

from __future__ import annotations

import ctypes
import functools
import threading
import time
from typing import Callable, Optional, Sequence

from . import _lib
from ._lib import check, ptr
from .concurrent_hash import LAUNCH_GEN as _MARK_GEN, BlockHashSet, BlockKey, CapacityExhausted, _as_keys
from .mc_encoding import FACE_BYTES, MC_BLOCK_BYTES, Q_BLOCK_BYTES, encode_keys, face_packs, pack_mc_batch
from .voxel_model import TSDF_BLOCK_BYTES

_MAX_SETS_PER_LAUNCH = 32


# One re-entrant lock for the server layer: its calls read and update host
# bookkeeping (FIFO ring bounds, the tables' last-launch streams, the tick's
# cached launch constants) around their launches, and the reference's Server
# calls these from several session threads (transport.py:157-160).  Launches
# stay asynchronous; only the host-side sequence is serialised, which costs
# nothing measurable (the calls are host-bound under the GIL anyway,
# DESIGN.md section 1).
_LOCK = threading.RLock()


def _locked(fn):
    @functools.wraps(fn)
    def wrapper(*a, **kw):
        with _LOCK:
            return fn(*a, **kw)

    return wrapper


class StreamSet:
    """Per-destination pending-update set with a generation-order queue
    (server.py:49-95).  The queue is a device ring of keys that keeps stale
    entries exactly like the reference's deque; ``extract_ordered`` skips
    them by validating membership.  The ring tail lives on the device so
    fan-outs need no host synchronisation; the host keeps the head and an
    upper bound of the tail for ring sizing."""

    def __init__(self, buckets: int = 1 << 16, excess: int = 1 << 16, *, device=None,
                 fifo_capacity: Optional[int] = None) -> None:
        torch = _lib.require_cuda()
        self._torch = torch
        self._set = BlockHashSet(buckets, excess, device=device)
        self.device = self._set.device
        cap = fifo_capacity or max(1024, min(buckets + excess, 1 << 20))
        self._fifo = torch.empty((cap, 3), dtype=torch.int32, device=self.device)
        self._head = 0
        self._tail_dev = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._tail_bound = 0
        self._scratch: Optional[BlockHashSet] = None

    def _grow(self, need: int = 0) -> None:
        """Lift the reference's fixed set capacity (server.py:242-243 caps a
        client's set at 2^16 + 2^16 and raises CapacityExhausted on larger
        models): move the pending keys into a table at least twice as large.
        The FIFO ring holds key values, so it stays as it is."""
        old = self._set
        nb, ex = 2 * old.bucket_count, 2 * old.excess_capacity
        while nb + ex < 2 * need:
            nb, ex = 2 * nb, 2 * ex
        keys, _ = old.snapshot_tensor()
        new = BlockHashSet(nb, ex, device=self.device)
        if keys.shape[0]:
            new.insert_keys(keys)
        new.check_capacity()
        self._set = new
        _FIFO_GEN[0] += 1  # cached launch arguments hold the old table

    # -- FIFO ring management -------------------------------------------------

    @property
    def fifo_capacity(self) -> int:
        return self._fifo.shape[0]

    def _tail(self) -> int:
        """Exact tail (synchronises with the table's stream)."""
        s = _order_streams([self._set])
        with self._torch.cuda.stream(s):
            t = int(self._tail_dev.item())
        self._tail_bound = t
        return t

    def _ring_view(self):
        """Pending FIFO entries [head, tail) in order (device tensor)."""
        torch = self._torch
        cap = self.fifo_capacity
        idx = torch.arange(self._head, self._tail(), device=self.device) % cap
        return self._fifo[idx]

    def _ensure_fifo(self, extra: int) -> None:
        if self._tail_bound + extra - self._head <= self.fifo_capacity:
            return
        tail = self._tail()
        need = tail - self._head + extra
        if need <= self.fifo_capacity:
            return
        torch = self._torch
        cap = max(2 * self.fifo_capacity, need)
        live = self._ring_view()
        fifo = torch.empty((cap, 3), dtype=torch.int32, device=self.device)
        fifo[: live.shape[0]] = live
        self._fifo = fifo
        _FIFO_GEN[0] += 1
        self._tail_dev.fill_(tail - self._head)
        self._tail_bound = tail - self._head
        self._head = 0

    @_locked
    def fifo_entries(self) -> list[BlockKey]:
        """The generation-order queue incl. stale entries (tests/inspection)."""
        return [tuple(k) for k in self._ring_view().cpu().tolist()]

    # -- reference API ------------------------------------------------------

    @_locked
    def insert(self, key: BlockKey) -> bool:
        return self.insert_many([key]) == 1

    @_locked
    def insert_many(self, keys) -> int:
        return fan_out([self], keys)[0]

    @_locked
    def remove(self, key: BlockKey) -> bool:
        return self._set.remove(key)

    @_locked
    def remove_many(self, keys) -> int:
        erased, _ = self._set.erase_keys(keys)
        return int(erased.sum().item())

    @_locked
    def size(self) -> int:
        return self._set.approx_size()

    @_locked
    def snapshot(self) -> list[BlockKey]:
        return self._set.snapshot_keys()

    @_locked
    def extract_random(self, max_n: int) -> list[BlockKey]:
        return self._set.extract_batch(max_n)

    @_locked
    def extract_matching(self, max_n: int, predicate: Callable) -> list[BlockKey]:
        return self._set.extract_matching(max_n, predicate)

    @_locked
    def extract_visible_first(self, max_n: int, planes, margin: float, block_size: float) -> list[BlockKey]:
        """VISIBLE_FIRST (server.py:339-344): frustum-visible keys first, then
        a random top-up so requests stay full-sized."""
        keys = self._set.extract_visible(max_n, planes, margin, block_size)
        if len(keys) < max_n:
            keys.extend(self.extract_random(max_n - len(keys)))
        return keys

    @_locked
    def extract_ordered(self, max_n: int) -> list[BlockKey]:
        keys = self.extract_ordered_keys(max_n)
        return [tuple(k) for k in keys.cpu().tolist()]

    @_locked
    def extract_ordered_keys(self, max_n: int):
        """Device version of extract_ordered (server.py:86-95) -> int32[m,3]."""
        torch = self._torch
        tail = self._tail()
        if max_n <= 0 or self._head >= tail:
            return torch.empty((0, 3), dtype=torch.int32, device=self.device)
        if self._scratch is None:
            self._scratch = BlockHashSet(1 << 12, 1 << 12, device=self.device)
        out = torch.empty((max_n, 3), dtype=torch.int32, device=self.device)
        head = ctypes.c_uint64(self._head)
        n_out = ctypes.c_uint64(0)
        s = _order_streams([self._set, self._scratch])
        check(_lib.load().vs_stream_extract_ordered(
            self._set.handle, ptr(self._fifo), self.fifo_capacity, ctypes.byref(head), tail, max_n,
            ptr(out), ctypes.byref(n_out), self._scratch.handle, ctypes.c_void_p(s.cuda_stream)),
            "extract_ordered")
        _mark_done([self._set, self._scratch], s)
        self._head = int(head.value)
        return out[: int(n_out.value)]

    @_locked
    def clear(self) -> None:
        """Bulk reset (fresh reconnect of a retained client)."""
        self._set.clear()
        s = _order_streams([self._set])
        with self._torch.cuda.stream(s):
            self._tail_dev.zero_()
        _mark_done([self._set], s)
        self._head = self._tail_bound = 0


def _order_streams(tables):
    """Current stream, ordered after the last launch on every table."""
    torch = tables[0]._torch
    s = torch.cuda.current_stream(tables[0].device)
    sid = s.cuda_stream
    for t in tables:
        if t._last_sid is not None and t._last_sid != sid:
            ev = torch.cuda.Event()
            ev.record(t._last_stream)
            s.wait_event(ev)
    return s


def _mark_done(tables, s) -> None:
    sid = s.cuda_stream
    for t in tables:
        t._last_stream = s
        t._last_sid = sid
    _MARK_GEN[0] += 1


# ctypes argument arrays of a client group, reused while the group's sets and
# FIFO rings are unchanged (a tick calls fan_out / extract on the same 16
# clients every time; rebuilding the arrays was a third of the host cost).
# Entries hold weak references, so a dead set never matches a new one.
_GROUP_CACHE: dict = {}
_FIFO_GEN = [0]  # bumped whenever a FIFO ring is reallocated


def _group_args(group):
    import weakref

    key = (tuple(map(id, group)), _FIFO_GEN[0])
    hit = _GROUP_CACHE.get(key)
    if hit is not None and all(r() is st for r, st in zip(hit[0], group)):
        return hit[1]
    C = len(group)
    tables = [st._set if isinstance(st, StreamSet) else st for st in group]
    args = {
        "tables": tables,
        "handles": (ctypes.c_void_p * C)(*[t.handle.value for t in tables]),
    }
    if all(isinstance(st, StreamSet) for st in group):
        args["fifos"] = (ctypes.c_void_p * C)(*[st._fifo.data_ptr() for st in group])
        args["caps"] = (ctypes.c_uint64 * C)(*[st.fifo_capacity for st in group])
        args["tails"] = (ctypes.c_void_p * C)(*[st._tail_dev.data_ptr() for st in group])
    if len(_GROUP_CACHE) >= 16:
        _GROUP_CACHE.clear()
    _GROUP_CACHE[key] = ([weakref.ref(st) for st in group], args)
    return args


@_locked
def fan_out(sets: Sequence[StreamSet], keys, *, sync: bool = True, n_dev=None):
    """``for s in sets: s.insert_many(keys)`` in one launch per 32 clients.

    For each client the newly created keys (the set difference keys \\
    pending) are appended to its FIFO in input order, exactly like the
    reference's per-key deque.append.  Returns the created count per client
    (synchronising), or the device counts (int64[C]) when sync=False.
    ``n_dev`` (device int64[1], optional): only the first min(n_dev, len(keys))
    keys count -- a device-produced count (vs_affected_dedup) needs no host
    synchronisation.
    """
    if not sets:
        return []
    torch = sets[0]._torch
    dev = sets[0].device
    k = _as_keys(keys, dev)
    n = k.shape[0]
    if n == 0:
        return [0] * len(sets) if sync else torch.zeros(len(sets), dtype=torch.int64, device=dev)
    lib = _lib.load()
    counts = torch.empty(len(sets), dtype=torch.int64, device=dev)
    created = torch.empty(min(len(sets), _MAX_SETS_PER_LAUNCH) * n, dtype=torch.uint8, device=dev)
    for g0 in range(0, len(sets), _MAX_SETS_PER_LAUNCH):
        group = sets[g0:g0 + _MAX_SETS_PER_LAUNCH]
        C = len(group)
        for st in group:
            if st._tail_bound + n - st._head > st._fifo.shape[0]:
                st._ensure_fifo(n)
        a = _group_args(group)
        tables = a["tables"]
        s = _order_streams(tables)
        check(lib.vs_stream_insert_many(a["handles"], C, ptr(k), n, ptr(n_dev), ptr(created), a["fifos"], a["caps"],
                                        a["tails"], ptr(counts[g0:g0 + C]), ctypes.c_void_p(s.cuda_stream)),
              "fan_out")
        _mark_done(tables, s)
        for st in group:
            st._tail_bound += n
    if not sync:
        return counts
    out = [int(c) for c in counts.cpu().tolist()]
    # a set that ran out of entries grows and takes the keys again (inserts of
    # keys it already holds are no-ops); sync=False callers check() instead
    for j, st in enumerate(sets):
        if isinstance(st, StreamSet):
            try:
                st._set.check_capacity()
            except CapacityExhausted:
                st._grow(st.size() + n)
                out[j] += fan_out([st], k)[0]
    return out


@_locked
def extract_random_many(sets: Sequence[StreamSet], max_n: int, seeds: Optional[Sequence[int]] = None, *,
                        n_out=None, keys_out=None):
    """``[s.extract_random(max_n) for s in sets]`` in one launch per 32
    clients.  Returns (keys int32[C, max_n, 3], n int64[C]) device tensors;
    ``n_out`` (optional device int64[C]) / ``keys_out`` (optional contiguous
    int32[C, max_n, 3]) receive the counts / keys instead of new tensors."""
    import random

    torch = sets[0]._torch
    dev = sets[0].device
    C = len(sets)
    if keys_out is not None:
        if keys_out.shape != (C, max(max_n, 1), 3) or keys_out.dtype != torch.int32 or not keys_out.is_contiguous():
            raise ValueError("keys_out must be a contiguous int32[C, max_n, 3] tensor")
        keys = keys_out
    else:
        keys = torch.empty((C, max(max_n, 1), 3), dtype=torch.int32, device=dev)
    n = n_out if n_out is not None else torch.empty(C, dtype=torch.int64, device=dev)
    if max_n <= 0:
        n.zero_()
        return keys[:, :0], n
    lib = _lib.load()
    for g0 in range(0, C, _MAX_SETS_PER_LAUNCH):
        group = sets[g0:g0 + _MAX_SETS_PER_LAUNCH]
        G = len(group)
        a = _group_args(group)
        tables = a["tables"]
        sd = (ctypes.c_uint64 * G)(*(seeds[g0:g0 + G] if seeds else [random.getrandbits(64) for _ in range(G)]))
        s = _order_streams(tables)
        check(lib.vs_stream_extract_random(a["handles"], G, max_n, sd, ptr(keys[g0:g0 + G]), ptr(n[g0:g0 + G]),
                                           ctypes.c_void_p(s.cuda_stream)), "extract_random_many")
        _mark_done(tables, s)
    return keys, n


@_locked
def stream_tick(sets: Sequence[StreamSet], updated, max_extract: int, seeds: Optional[Sequence[int]] = None, *,
                affected_out=None, n_affected=None, keys_out=None, n_out=None, n_created=None):
    """One tick of the server's stream-set path in ONE launch per 32 clients:
    the affected dedup of the updated TSDF keys (server.py:304-307), the
    fan-out of the affected keys into every client set with the FIFO append
    (server.py:314-315), and an extract_random(max_extract) per client
    (server.py:334-363) -- ``affected_dedup`` + ``fan_out`` +
    ``extract_random_many`` fused (k_stream_tick).  1 <= len(updated) <= 512.

    Returns (affected int32[8U,3], n_affected int64[1], keys int32[C,max_n,3],
    n int64[C]) device tensors (or the given ``*_out`` buffers); nothing
    synchronises."""
    import random

    torch = sets[0]._torch
    dev = sets[0].device
    k = _as_keys(updated, dev)
    U = k.shape[0]
    C = len(sets)
    if not 1 <= U <= 512:
        raise ValueError("stream_tick takes 1..512 updated keys (larger updates: affected_dedup + fan_out)")
    if C > _MAX_SETS_PER_LAUNCH:
        raise ValueError(f"stream_tick takes at most {_MAX_SETS_PER_LAUNCH} client sets per call")
    aff = affected_out if affected_out is not None else torch.empty((8 * U, 3), dtype=torch.int32, device=dev)
    na = n_affected if n_affected is not None else torch.empty(1, dtype=torch.int64, device=dev)
    X = max(max_extract, 1)
    keys = keys_out if keys_out is not None else torch.empty((C, X, 3), dtype=torch.int32, device=dev)
    n = n_out if n_out is not None else torch.empty(C, dtype=torch.int64, device=dev)
    for st in sets:
        if st._tail_bound + 8 * U - st._head > st._fifo.shape[0]:
            st._ensure_fifo(8 * U)
    a = _group_args(list(sets))
    tables = a["tables"]
    sd = (ctypes.c_uint64 * C)(*(seeds if seeds else [random.getrandbits(64) for _ in range(C)]))
    s = _order_streams(tables)
    check(_lib.load().vs_stream_tick(a["handles"], C, ptr(k), U, a["fifos"], a["caps"], a["tails"], max_extract, sd,
                                     ptr(aff), ptr(na), ptr(n_created), ptr(keys), ptr(n),
                                     ctypes.c_void_p(s.cuda_stream)), "stream_tick")
    _mark_done(tables, s)
    for st in sets:
        st._tail_bound += 8 * U
    return aff, na, keys, n


@_locked
def remove_everywhere(sets: Sequence[StreamSet], keys) -> None:
    """Remove keys from every client set (server.py:433-435), one launch per 32."""
    if not sets:
        return
    dev = sets[0].device
    k = _as_keys(keys, dev)
    if k.shape[0] == 0:
        return
    lib = _lib.load()
    for g0 in range(0, len(sets), _MAX_SETS_PER_LAUNCH):
        tables = [st._set for st in sets[g0:g0 + _MAX_SETS_PER_LAUNCH]]
        handles = (ctypes.c_void_p * len(tables))(*[t.handle.value for t in tables])
        s = _order_streams(tables)
        check(lib.vs_stream_remove_many(handles, len(tables), ptr(k), k.shape[0], None,
                                        ctypes.c_void_p(s.cuda_stream)), "remove_everywhere")
        _mark_done(tables, s)


class GpuServerCore:
    """Device-resident TSDF model, MC model and client stream sets.

    tsdf_map / mc_map are hash tables whose entry positions index the device
    payload pools (the reference's parallel ``_values`` array,
    concurrent_hash.py:112): tsdf_pool uint8[cap,6144] (wire rows),
    mc_pool uint8[cap,2048] (McBlock.to_bytes), q_pool int8[cap,512].
    tsdf_faces uint8[cap,48] holds the face bit-packs of the TSDF rows (the
    encoder's halo side table), refreshed for every row the ingest writes.
    """

    def __init__(self, buckets: int = 1 << 20, excess: int = 1 << 20, *, stream_buckets: int = 1 << 16,
                 stream_excess: int = 1 << 16, retention_s: float = 3600.0, max_batch: int = 4096,
                 device=None) -> None:
        torch = _lib.require_cuda()
        self._torch = torch
        self.tsdf_map = BlockHashSet(buckets, excess, device=device)
        self.device = self.tsdf_map.device
        self.mc_map = BlockHashSet(buckets, excess, device=self.device)
        cap = buckets + excess
        self.tsdf_pool = torch.zeros((cap, TSDF_BLOCK_BYTES), dtype=torch.uint8, device=self.device)
        self.tsdf_faces = torch.zeros((cap, FACE_BYTES), dtype=torch.uint8, device=self.device)
        self.mc_pool = torch.zeros((cap, MC_BLOCK_BYTES), dtype=torch.uint8, device=self.device)
        self.q_pool = torch.zeros((cap, Q_BLOCK_BYTES), dtype=torch.int8, device=self.device)
        self._dedup = BlockHashSet(16 * max_batch, 16 * max_batch, device=self.device)
        self._tick_cache = None  # on_tsdf_batch(sync=False) per-group launch constants
        self._stream_sizes = (stream_buckets, stream_excess)
        self.retention_s = retention_s
        self.sessions: dict[bytes, dict] = {}

    # -- sessions (server.py:221-249) ---------------------------------------

    @_locked
    def attach(self, client_id: bytes) -> StreamSet:
        """Returning client within retention keeps its set; otherwise a new
        set filled with every MC key (snapshot order)."""
        now = time.monotonic()
        sess = self.sessions.get(client_id)
        if sess is not None and (sess["connected"] or now - sess["disconnected_at"] <= self.retention_s):
            sess["connected"] = True
            return sess["stream"]
        stream = StreamSet(*self._stream_sizes, device=self.device)
        self.sessions[client_id] = {"stream": stream, "connected": True, "disconnected_at": 0.0}
        keys, _ = self.mc_map.snapshot_tensor()
        fan_out([stream], keys)
        return stream

    @_locked
    def detach(self, client_id: bytes) -> None:
        sess = self.sessions.get(client_id)
        if sess is not None:
            sess["connected"] = False
            sess["disconnected_at"] = time.monotonic()

    def streams(self) -> list[StreamSet]:
        return [s["stream"] for s in self.sessions.values()]

    # -- model updates (server.py:299-315) ----------------------------------

    @_locked
    def on_tsdf_batch(self, keys, rows, *, sync: bool = True):
        """Ingest U TSDF blocks (int32[U,3], uint8[U,6144] wire rows) and
        propagate (server.py:299-315): TSDF put (latest write wins), face
        packs of the written rows, affected = ordered first-occurrence dedup
        of the 8 affected MC keys per block, mc_map.put + recompute (the
        encoder writes straight into mc_pool / q_pool at the MC map
        positions), insert_many into every client set.

        sync=True keeps the reference's exact failure semantics (a put that
        finds the excess list empty raises CapacityExhausted with the earlier
        blocks applied) and returns the affected keys (device int32[A,3]).
        sync=False queues the whole update with NO host synchronisation (the
        device-side affected count bounds every later launch) and returns
        (affected int32[8U,3], n_affected int64[1]) device tensors; a
        capacity failure is sticky and raised by ``check()``."""
        torch = self._torch
        dev = self.device
        k = _as_keys(keys, dev)
        if not (isinstance(rows, torch.Tensor) and rows.dtype == torch.uint8 and rows.device == dev):
            rows = torch.as_tensor(rows).to(dev, torch.uint8)
        rows = rows.reshape(-1, TSDF_BLOCK_BYTES)
        U = k.shape[0]
        if U == 0:
            return k if sync else (k, torch.zeros(1, dtype=torch.int64, device=dev))
        lib = _lib.load()
        if 8 * U > self._dedup.bucket_count:
            self._dedup = BlockHashSet(16 * U, 16 * U, device=dev)
        if not sync:
            # the whole chain in ONE host call (vs_server_tick): the per-call
            # host work of the separate calls below was the tick's critical path
            rows = rows.contiguous()
            # one allocation for both outputs (views), raw pointers as ints:
            # this wrapper's own cost is part of the tick when the host paces it
            out = torch.empty(24 * U + 2, dtype=torch.int32, device=dev)
            affected = out[: 24 * U].view(8 * U, 3)
            n_dev = out[24 * U:].view(torch.int64)
            streams = self.streams()
            need = 8 * U
            # per-tick constants of this client group (tables, ctypes arrays,
            # pool pointers, ring capacities), rebuilt when the group, a ring
            # or a table changes
            key = (tuple(map(id, streams)), _FIFO_GEN[0], id(self._dedup))
            tc = self._tick_cache
            caps = tc["caps"] if tc is not None and tc["key"] == key else [st.fifo_capacity for st in streams]
            for st, cap in zip(streams, caps):
                if st._tail_bound + need - st._head > cap:
                    st._ensure_fifo(need)  # may reallocate the ring (bumps _FIFO_GEN: the key below changes)
            key = (key[0], _FIFO_GEN[0], key[2])
            if tc is None or tc["key"] != key:
                a = _group_args(streams) if streams else None
                tc = self._tick_cache = {
                    "key": key, "tables": [self.tsdf_map, self.mc_map, self._dedup] + (a["tables"] if a else []),
                    "caps": [st.fifo_capacity for st in streams], "mark": None, "sid": None,
                    "args": (self.tsdf_map.handle, self.mc_map.handle, self._dedup.handle),
                    "pools": (self.tsdf_pool.data_ptr(), self.tsdf_faces.data_ptr(), self.mc_pool.data_ptr(),
                              self.q_pool.data_ptr()),
                    "group": (a["handles"] if a else None, len(streams), a["fifos"] if a else None,
                              a["caps"] if a else None, a["tails"] if a else None)}
            cur = torch.cuda.current_stream(dev)
            sid = cur.cuda_stream
            if tc["mark"] == _MARK_GEN[0] and tc["sid"] == sid:
                s = cur  # back to back with this core's previous tick on the same stream: already ordered
            else:
                s = _order_streams(tc["tables"])
            t0, t1, t2 = tc["args"]
            p0, p1, p2, p3 = tc["pools"]
            g0, g1, g2, g3, g4 = tc["group"]
            check(lib.vs_server_tick(t0, t1, t2, k.data_ptr(), rows.data_ptr(), U, p0, p1, p2, p3, g0, g1, g2, g3,
                                     g4, affected.data_ptr(), n_dev.data_ptr(), sid), "server_tick")
            if tc["mark"] != _MARK_GEN[0] or tc["sid"] != sid:
                _mark_done(tc["tables"], s)
                tc["mark"], tc["sid"] = _MARK_GEN[0], sid
            for st in streams:
                st._tail_bound += need
            return affected, n_dev
        # exact sequential failure semantics first (the reference raises at
        # the first block that finds the excess list empty)
        self.tsdf_map.insert_many_exact(k)
        pos = torch.empty(U, dtype=torch.int32, device=dev)
        rows = rows.contiguous()
        st = _order_streams([self.tsdf_map])
        check(lib.vs_tsdf_put(self.tsdf_map.handle, ptr(k), ptr(rows), U, ptr(self.tsdf_pool), ptr(pos),
                              ctypes.c_void_p(st.cuda_stream)), "tsdf_put")
        _mark_done([self.tsdf_map], st)
        face_packs(self.tsdf_pool, rows=pos, faces=self.tsdf_faces)  # halo side table of the written rows
        affected = torch.empty((8 * U, 3), dtype=torch.int32, device=dev)
        n_dev = torch.empty(1, dtype=torch.int64, device=dev)
        s = _order_streams([self._dedup])
        check(lib.vs_affected_dedup(self._dedup.handle, ptr(k), U, ptr(affected), ptr(n_dev),
                                    ctypes.c_void_p(s.cuda_stream)), "affected_dedup")
        _mark_done([self._dedup], s)
        A = int(n_dev.item())
        affected = affected[:A]
        _, mpos = self.mc_map.insert_many_exact(affected)  # mc_map.put (positions of every key)
        # recompute straight into the MC / quantised pools at the map positions
        encode_keys(self.tsdf_map, self.tsdf_pool, affected, mc=self.mc_pool, q=self.q_pool, counts=False,
                    faces=self.tsdf_faces, out_rows=mpos)
        streams = self.streams()
        if streams:
            fan_out(streams, affected, sync=False)
        return affected

    @_locked
    def check(self) -> None:
        """Raise CapacityExhausted if a sync=False update ran out of entries
        (in either map or in a client's stream set)."""
        self.tsdf_map.check_capacity()
        self.mc_map.check_capacity()
        for st in self.streams():
            st._set.check_capacity()

    @_locked
    def on_reset_blocks(self, keys) -> None:
        """server.py:425-436: remove from both maps and every client set."""
        k = _as_keys(keys, self.device)
        if k.shape[0] == 0:
            return
        _, tpos = self.tsdf_map.erase_keys(k)
        _, mpos = self.mc_map.erase_keys(k)
        remove_everywhere(self.streams(), k)

    @_locked
    def on_block_request(self, client_id: bytes, max_blocks: int, strategy: int, planes=None,
                         margin: float = 0.0, block_size: float = 0.04) -> tuple[list, bytes]:
        """server.py:334-363 without the transport: extract by strategy
        (0 GENERATION_ORDER, 1 VISIBLE_FIRST, 2 RANDOM), drop keys deleted
        meanwhile, and pack the MC_BATCH payload (wire.py:292-299) from the
        device MC pool.  Returns (keys, payload bytes)."""
        torch = self._torch
        st = self.sessions[client_id]["stream"]
        if strategy == 1:
            keys = st.extract_visible_first(max_blocks, planes, margin, block_size)
        elif strategy == 0:
            keys = st.extract_ordered(max_blocks)
        else:
            keys = st.extract_random(max_blocks)
        if not keys:
            return [], (0).to_bytes(4, "little")
        k = _as_keys(keys, self.device)
        found, pos = self.mc_map.find_keys(k)
        keep = found.bool()
        payload = pack_mc_batch(k[keep], pos[keep], self.mc_pool)
        kept = [kk for kk, f in zip(keys, found.cpu().tolist()) if f]
        return kept, bytes(payload.cpu().numpy().tobytes())

    @_locked
    def mc_payload(self, key: BlockKey) -> Optional[bytes]:
        found, pos = self.mc_map.find_keys([key])
        if not bool(found[0].item()):
            return None
        return bytes(self.mc_pool[int(pos[0].item())].cpu().numpy().tobytes())

    @_locked
    def tsdf_payload(self, key: BlockKey) -> Optional[bytes]:
        found, pos = self.tsdf_map.find_keys([key])
        if not bool(found[0].item()):
            return None
        return bytes(self.tsdf_pool[int(pos[0].item())].cpu().numpy().tobytes())
