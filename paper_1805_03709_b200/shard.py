"""Key-hash sharded block hash set across GPUs.

Every rank owns one partition of the key space: owner(k) = fmix32(h(k)) mod
G, where h is the reference's pre-modulo spatial hash (concurrent_hash.py:58)
and fmix32 (MurmurHash3 finaliser) decorrelates the owner from the local
bucket h mod n.

Two exchanges route a batch to the owners and back.

``exchange="peer"`` (the product path on GPUs; csrc/shard.cu): every rank
maps every other rank's receive window over CUDA IPC (NVLink/NVSwitch), and
the kernels themselves store each op's 16-byte record into its owner's
window, apply the owner's ops, and store each result byte back into the
source's window -- one stream-ordered call per batch, no host
synchronisation, no NCCL.  The windows are exchanged once, at construction,
over the process group.

``exchange="collective"`` (the parity reference for the peer path, and the
CPU/gloo path of the multi-process tests):

  1. owner of every op, stable partition of the batch by owner
  2. all-to-all of the per-owner counts
  3. all-to-all of 16-byte records {x, y, z, op}
  4. one local ``apply`` launch on the owned table (vs_table_apply)
  5. all-to-all of the 1-byte results back, scatter to the input order

Over NCCL the exchanges run on NVLink/NVSwitch; the same code runs over gloo
on CPU for the multi-process tests.  A18 batches stay order-independent
under routing, so per-op results are still bit-exact with a sequential
replay of the union of all ranks' batches.
"""

from __future__ import annotations

from typing import Optional


def owner_of(keys, world: int):
    """fmix32(hash_key pre-modulo) mod world, on int32[N,3] tensors."""
    import torch

    k = keys.to(torch.int64)
    h = ((k[:, 0] * 73856093) ^ (k[:, 1] * 19349669) ^ (k[:, 2] * 83492791)) & 0xFFFFFFFF
    h = ((h ^ (h >> 16)) * 0x85EBCA6B) & 0xFFFFFFFF
    h = ((h ^ (h >> 13)) * 0xC2B2AE35) & 0xFFFFFFFF
    h = h ^ (h >> 16)
    return h % world


class ShardedBlockHashSet:
    """A block hash set partitioned over the ranks of a process group.

    ``local`` is the rank's own table (a BlockHashSet on its GPU; tests may
    pass any object with the same ``apply`` signature).  ``exchange``:
    "peer" (kernel peer stores over CUDA IPC windows; needs a BlockHashSet
    on a CUDA device), "collective" (all-to-all over the process group), or
    "auto" (peer when the local table is a device table, else collective).
    ``max_batch`` bounds the ops per ``apply`` call on the peer path (it
    sizes the windows: world x max_batch x 16 B per rank).
    """

    def __init__(self, local, group=None, exchange: str = "auto", max_batch: int = 1 << 22) -> None:
        import torch.distributed as dist

        if exchange not in ("auto", "peer", "collective"):
            raise ValueError(f"unknown exchange {exchange!r}")
        self.local = local
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)
        self._stage = False
        self._shard = None
        self.max_batch = int(max_batch)
        device_table = getattr(local, "handle", None) is not None and getattr(local, "device", None) is not None \
            and getattr(local.device, "type", None) == "cuda"
        if exchange == "peer" and not device_table:
            raise ValueError("exchange='peer' needs a BlockHashSet on a CUDA device")
        self.exchange = "peer" if (exchange == "peer" or (exchange == "auto" and device_table)) else "collective"
        if self.exchange == "peer" and not self._connect(required=exchange == "peer"):
            self.exchange = "collective"

    # -- peer-window exchange (csrc/shard.cu) ------------------------------

    def _connect(self, required: bool) -> bool:
        """Create this rank's window, exchange the IPC handles, map the peers.
        Collective.  Every rank learns whether ALL ranks succeeded; when one
        did not (e.g. no peer access between two GPUs) and the peer route was
        not required, every rank falls back to the collective route together."""
        import ctypes
        import warnings

        import torch
        import torch.distributed as dist

        from . import _lib

        lib = _lib.load()
        self._lib = lib
        mine = (ctypes.c_uint8 * 64)()
        err = ""
        try:
            h = ctypes.c_void_p()
            _lib.check(lib.vs_shard_create(self.local.handle, self.rank, self.world, self.max_batch,
                                           ctypes.byref(h)), "vs_shard_create")
            self._shard = h
            _lib.check(lib.vs_shard_export(h, ctypes.byref(mine)), "vs_shard_export")
        except Exception as exc:  # noqa: BLE001 - reported below, decided collectively
            err = str(exc)
        handles: list = [None] * self.world
        dist.all_gather_object(handles, None if err else bytes(mine), group=self.group)
        if not err and all(x is not None for x in handles):
            try:
                _lib.check(lib.vs_shard_connect(self._shard, b"".join(handles)), "vs_shard_connect")
            except Exception as exc:  # noqa: BLE001
                err = str(exc)
        elif not err:
            err = "a peer could not create its window"
        ok = torch.tensor([0 if err else 1], dtype=torch.int32)
        if self.backend == "nccl":
            ok = ok.to(self.local.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if int(ok.item()) == 0:
            if self._shard is not None:
                lib.vs_shard_destroy(self._shard)
                self._shard = None
            if required:
                raise RuntimeError(f"peer route unavailable: {err or 'failed on another rank'}")
            warnings.warn(f"peer route unavailable ({err or 'failed on another rank'}); using the collective route")
            return False
        # every rank mapped every window before anyone stores into one
        dist.barrier(group=self.group)
        return True

    def __del__(self) -> None:
        h = getattr(self, "_shard", None)
        if h is not None and h.value:
            try:
                self._lib.vs_shard_destroy(h)
            except Exception:
                pass
            self._shard = None

    def check(self) -> None:
        """Raise if a peer wait timed out (mismatched collective calls)."""
        if self._shard is not None:
            from . import _lib

            _lib.check(self._lib.vs_shard_check(self._shard), "vs_shard")

    def _apply_peer(self, keys, ops):
        import ctypes

        import torch

        from . import _lib

        loc = self.local
        n = keys.shape[0]
        if n > self.max_batch:
            raise ValueError(f"batch of {n} ops exceeds max_batch={self.max_batch} of the shard windows")
        with loc._mutex:
            k = loc._keys(keys)
            o = ops.to(loc.device, torch.uint8).contiguous()
            if o.shape[0] != n:
                raise ValueError("ops and keys differ in length")
            out = torch.empty(n, dtype=torch.uint8, device=loc.device)
            s = loc._stream()
            _lib.check(self._lib.vs_shard_apply(self._shard, _lib.ptr(k), _lib.ptr(o), n, _lib.ptr(out),
                                                ctypes.c_void_p(s.cuda_stream)), "vs_shard_apply")
            loc._done(s)
        return out

    def _a2a(self, out, inp, out_splits=None, in_splits=None):
        """all_to_all_single; staged through host memory when the backend
        cannot move device tensors (gloo: multi-rank tests on one GPU)."""
        import torch.distributed as dist

        if self._stage:
            o = out.cpu()
            dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=self.group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def apply(self, keys, ops, device: Optional[object] = None):
        """Mixed batch (ops 0 insert / 1 find / 2 erase) of THIS rank; returns
        the per-op results in input order.  Collective: every rank calls it."""
        import torch

        if self.exchange == "peer":
            return self._apply_peer(keys, ops)
        dev = keys.device
        self._stage = dev.type == "cuda" and self.backend == "gloo"
        own = owner_of(keys, self.world)
        order = torch.argsort(own, stable=True)
        send_counts = torch.bincount(own, minlength=self.world)
        recv_counts = torch.empty_like(send_counts)
        self._a2a(recv_counts, send_counts)
        sc, rc = send_counts.tolist(), recv_counts.tolist()
        payload = torch.cat([keys[order].to(torch.int32), ops[order].to(torch.int32)[:, None]], dim=1).contiguous()
        recv = torch.empty((sum(rc), 4), dtype=torch.int32, device=dev)
        self._a2a(recv, payload, rc, sc)
        res, _ = self.local.apply(recv[:, :3].contiguous(), recv[:, 3].to(torch.uint8))
        back = torch.empty(keys.shape[0], dtype=torch.uint8, device=dev)
        self._a2a(back, res.to(torch.uint8).contiguous(), sc, rc)
        out = torch.empty_like(back)
        out[order] = back
        return out

    def size(self) -> int:
        import torch
        import torch.distributed as dist

        n = torch.tensor([self.local.approx_size()], dtype=torch.int64)
        if self.backend == "nccl":
            n = n.cuda()
        dist.all_reduce(n, group=self.group)
        return int(n.item())


class OneGpuShardGroup:
    """All `world` ranks of a sharded set on ONE GPU in ONE process (tests and
    diagnostics): rank r owns `tables[r]`; ``apply`` queues every rank's
    batch on the rank's own stream, exactly as G processes would, and the
    kernels route through the same windows and flags as across GPUs
    (csrc/shard.cu, vs_shard_connect_local).  The process must give every
    rank stream its own hardware queue (CUDA_DEVICE_MAX_CONNECTIONS >= world
    + 1, set before CUDA initialises), or a rank's push can queue behind
    another rank's spin-wait; such a wait times out and check() raises."""

    def __init__(self, tables, max_batch: int) -> None:
        import ctypes

        import torch

        from . import _lib

        self._lib = _lib.load()
        self.tables = list(tables)
        self.world = len(self.tables)
        self.max_batch = int(max_batch)
        self.device = self.tables[0].device
        self.shards = []
        for r, t in enumerate(self.tables):
            h = ctypes.c_void_p()
            _lib.check(self._lib.vs_shard_create(t.handle, r, self.world, self.max_batch, ctypes.byref(h)),
                       "vs_shard_create")
            self.shards.append(h)
        arr = (ctypes.c_void_p * self.world)(*[h.value for h in self.shards])
        _lib.check(self._lib.vs_shard_connect_local(arr, self.world), "vs_shard_connect_local")
        self.streams = [torch.cuda.Stream(self.device) for _ in range(self.world)]

    def apply(self, keys_list, ops_list):
        """One collective batch: keys_list[r] / ops_list[r] are rank r's ops;
        returns the per-rank results (device uint8), ordered after the call."""
        import ctypes

        import torch

        from . import _lib

        cur = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(cur)
        outs = []
        for r in range(self.world):
            k = keys_list[r].to(self.device, torch.int32).contiguous()
            o = ops_list[r].to(self.device, torch.uint8).contiguous()
            out = torch.empty(k.shape[0], dtype=torch.uint8, device=self.device)
            st = self.streams[r]
            st.wait_event(ev)
            k.record_stream(st)
            o.record_stream(st)
            out.record_stream(st)
            _lib.check(self._lib.vs_shard_apply(self.shards[r], _lib.ptr(k), _lib.ptr(o), k.shape[0], _lib.ptr(out),
                                                ctypes.c_void_p(st.cuda_stream)), "vs_shard_apply")
            outs.append(out)
        for st in self.streams:
            cur.wait_stream(st)
        return outs

    def check(self) -> None:
        from . import _lib

        for h in self.shards:
            _lib.check(self._lib.vs_shard_check(h), "vs_shard")

    def __del__(self) -> None:
        for h in getattr(self, "shards", []):
            try:
                self._lib.vs_shard_destroy(h)
            except Exception:
                pass
        self.shards = []
