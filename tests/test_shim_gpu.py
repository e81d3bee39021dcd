"""The drop-in boundary end to end: the reference Server's on_tsdf_batch as
installed by ``shim.install()`` (shim._on_tsdf_batch), driven on the GPU
tables / stream sets with the reference's recorded 3-client server sequence
(tests/golden/server_seq.json, server_blocks.npz: gen_golden.py replays
voxelstream.server.Server and records every client's FIFO appends, pending
sets, MC payload digests and the fresh-attach fill).

The reference package is not on the GPU box, so the Server is a stub that
carries exactly the attributes the reference methods touch
(server.py:221-249, 299-323, 425-436): ``tsdf_map`` / ``mc_map``
(BlockHashMap), ``sessions`` with ``.stream`` per exploration client,
``_exploration_sessions()``; ``_attach_session`` and ``on_reset_blocks``
are the reference's own statements (fresh branch / the removal loops) over
the GPU objects.
"""

from __future__ import annotations

import hashlib
import json
import sys

import numpy as np
import pytest

from paper_1805_03709_b200.voxel_model import TsdfBlock  # noqa: F401  (read by shim._on_tsdf_batch)

pytestmark = pytest.mark.gpu


class _Batch:
    def __init__(self, blocks):
        self.blocks = blocks  # [(key, 6144 raw bytes)] as wire.TsdfBatch.blocks


class _Session:
    def __init__(self, stream):
        self.stream = stream


class StubServer:
    """The reference Server's state used by on_tsdf_batch (server.py:299-323)."""

    def __init__(self):
        from paper_1805_03709_b200 import BlockHashMap

        self.tsdf_map = BlockHashMap(1 << 12, 1 << 12)
        self.mc_map = BlockHashMap(1 << 12, 1 << 12)
        self.sessions = {}

    def _exploration_sessions(self):
        return list(self.sessions.values())

    def _attach_session(self, client_id):
        """The fresh-client branch of server.py:240-248."""
        from paper_1805_03709_b200 import StreamSet

        stream = StreamSet(1 << 10, 1 << 10)
        stream.insert_many(self.mc_map.snapshot_keys())
        self.sessions[client_id] = _Session(stream)
        return stream

    def on_reset_blocks(self, keys):
        """server.py:425-436 (without the DeleteBlocks send)."""
        for key in keys:
            self.tsdf_map.remove(key)
            self.mc_map.remove(key)
        for ec in self._exploration_sessions():
            for key in keys:
                ec.stream.remove(key)


def test_shim_on_tsdf_batch_replays_reference_server(dev, golden):
    from paper_1805_03709_b200 import shim

    assert sys.modules[StubServer.__module__].TsdfBlock is TsdfBlock
    g = json.loads((golden / "server_seq.json").read_text())
    d = np.load(golden / "server_blocks.npz")
    srv = StubServer()
    clients = [srv._attach_session(bytes([i]) * 16) for i in range(3)]
    for step, entry in enumerate(g["steps"]):
        sel = d["step"] == step
        keys = [tuple(int(v) for v in k) for k in d["keys"][sel]]
        assert [list(k) for k in keys] == entry["updated"]
        batch = _Batch([(k, bytes(b.tobytes())) for k, b in zip(keys, d["blocks"][sel])])
        before = [len(c.fifo_entries()) for c in clients]
        shim._on_tsdf_batch(srv, batch)
        for c, cl in enumerate(clients):
            assert [list(k) for k in cl.fifo_entries()[before[c]:]] == entry["appended"][c]
            assert sorted(list(k) for k in cl.snapshot()) == entry["pending"][c]
        if "pending_after_extract_c1" in entry:
            keep = {tuple(k) for k in entry["pending_after_extract_c1"]}
            drop = [k for k in clients[1].snapshot() if k not in keep]
            clients[1].remove_many(drop)  # adopt the reference's random subset
        if "reset" in entry:
            srv.on_reset_blocks([tuple(v) for v in entry["reset"]])
            for c, cl in enumerate(clients):
                assert sorted(list(k) for k in cl.snapshot()) == entry["pending_after_reset"][c]
    got = sorted(srv.mc_map.snapshot_keys())
    assert [list(k) for k in got] == g["mc_keys"]
    for k in got:  # MC payloads stored pre-serialised, as server.py:312-313
        assert hashlib.sha256(srv.mc_map.get(k)).hexdigest() == g["mc_digest"][",".join(map(str, k))], k
    fresh = srv._attach_session(b"\x09" * 16)
    assert sorted(list(k) for k in fresh.snapshot()) == g["fresh_pending"]


def test_gpu_server_core_sync_free_tick_matches_sync(dev, golden):
    """GpuServerCore.on_tsdf_batch(sync=False) -- the host-sync-free tick --
    leaves the same MC pool bytes, quantised bytes and client FIFOs as the
    exact (sync=True) path on the reference sequence."""
    import torch

    from paper_1805_03709_b200 import GpuServerCore

    g = json.loads((golden / "server_seq.json").read_text())
    d = np.load(golden / "server_blocks.npz")
    cores = [GpuServerCore(1 << 12, 1 << 12, stream_buckets=1 << 10, stream_excess=1 << 10) for _ in range(2)]
    cl = [[core.attach(bytes([i]) * 16) for i in range(3)] for core in cores]
    for step, entry in enumerate(g["steps"]):
        sel = d["step"] == step
        a0 = cores[0].on_tsdf_batch(d["keys"][sel], d["blocks"][sel])
        a1, n1 = cores[1].on_tsdf_batch(d["keys"][sel], d["blocks"][sel], sync=False)
        assert torch.equal(a0, a1[: int(n1.item())])
        cores[1].check()
        for c in range(3):  # core 0 (exact path) is checked against the reference in test_stream_gpu
            assert cl[0][c].fifo_entries() == cl[1][c].fifo_entries()
            assert sorted(list(k) for k in cl[1][c].snapshot()) == entry["pending"][c]
        if "pending_after_extract_c1" in entry:
            keep = {tuple(k) for k in entry["pending_after_extract_c1"]}
            for core_cl in cl:
                core_cl[1].remove_many([k for k in core_cl[1].snapshot() if k not in keep])
        if "reset" in entry:
            for core in cores:
                core.on_reset_blocks([tuple(v) for v in entry["reset"]])
    for k in g["mc_keys"]:
        k = tuple(k)
        assert hashlib.sha256(cores[1].mc_payload(k)).hexdigest() == g["mc_digest"][",".join(map(str, k))], k
        f0, p0 = cores[0].mc_map.find_keys([k])
        f1, p1 = cores[1].mc_map.find_keys([k])
        assert torch.equal(cores[0].q_pool[p0.long()], cores[1].q_pool[p1.long()])
