"""Key-hash sharded block hash set across GPUs.

Every rank owns one partition of the key space: owner(k) = fmix32(h(k)) mod
G, where h is the reference's pre-modulo spatial hash (concurrent_hash.py:58)
and fmix32 (MurmurHash3 finaliser) decorrelates the owner from the local
bucket h mod n.  A batch is routed to the owners and back:

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
    pass any object with the same ``apply`` signature).
    """

    def __init__(self, local, group=None) -> None:
        import torch.distributed as dist

        self.local = local
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)
        self._stage = False

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
