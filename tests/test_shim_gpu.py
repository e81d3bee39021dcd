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
import threading
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
        self.sent = []

    def send(self, msg, codec):
        self.sent.append(msg.keys)
        return True


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


@pytest.mark.parametrize("batched_reset", [False, True])
def test_shim_on_tsdf_batch_replays_reference_server(dev, golden, batched_reset):
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
            if batched_reset:  # shim._on_reset_blocks: batched removes + DeleteBlocks to each client
                srv.cfg = _types.SimpleNamespace(codec=None)
                srv._delivery_lock = threading.Lock()
                shim._on_reset_blocks(srv, [tuple(v) for v in entry["reset"]])
                assert all(s_.sent and s_.sent[-1] == [tuple(v) for v in entry["reset"]]
                           for s_ in srv.sessions.values())
            else:
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


# ---- on_block_request through the shim: the names server.py imports, stubbed
# (the reference package is not on the GPU box)
import enum as _enum
import types as _types


class _Strategy(_enum.IntEnum):
    GENERATION_ORDER = 0
    VISIBLE_FIRST = 1
    RANDOM = 2


class _McBatch:
    def __init__(self, blocks):
        self.blocks = blocks


class _DeleteBlocks:
    def __init__(self, keys):
        self.keys = keys


wire = _types.SimpleNamespace(Strategy=_Strategy, McBatch=_McBatch, DeleteBlocks=_DeleteBlocks)
BLOCK_EDGE = 8


class Pose:
    @staticmethod
    def from_floats(v):
        return tuple(v)


class CameraIntrinsics:
    def __init__(self, **kw):
        self.kw = kw


class Frustum:
    """Stand-in with the two attributes the predicate uses: the half-space
    x >= 0.2 (plus five planes every block passes)."""

    def __init__(self, pose, intr, near, far, margin):
        self.margin = margin
        self._planes = [(1.0, 0.0, 0.0, -0.2)] + [(0.0, 0.0, 0.0, 1.0)] * 5


class _Sess:
    def __init__(self, stream):
        self.stream = stream
        self.request_count = self.blocks_sent = 0
        self.sent = []

    def send(self, msg, codec):
        self.sent.append(msg.blocks)
        return True


def test_shim_block_request_device_frustum_and_batched_gets(dev):
    """VISIBLE_FIRST through shim._on_block_request on a GPU stream set: the
    frustum from the request goes to the device predicate (visible keys
    first, random top-up), payloads come from ONE batched map lookup, keys
    deleted from the map meanwhile are dropped."""
    import threading

    from paper_1805_03709_b200 import BlockHashMap, StreamSet, shim

    srv = StubServer()
    srv.mc_map = BlockHashMap(1 << 10, 1 << 10)
    srv.cfg = _types.SimpleNamespace(max_request_blocks=64, codec=None, voxel_size=0.01)
    srv._delivery_lock = threading.Lock()
    keys = [(x, y, 0) for x in range(-8, 8) for y in range(4)]  # 64 keys; x >= 0 is visible with block 0.08
    for k in keys:
        srv.mc_map.put(k, bytes([k[0] & 0xFF, k[1]]))
    srv.mc_map.remove((5, 1, 0))  # deleted by a reset after it became pending
    stream = StreamSet(1 << 8, 1 << 8)
    stream.insert_many(keys)
    sess = _Sess(stream)
    req = _types.SimpleNamespace(max_blocks=40, strategy=_Strategy.VISIBLE_FIRST, intrinsics=(1.0, 1.0, 320.0, 240.0,
                                 0.1, 10.0), pose=(0.0,) * 7)
    shim._on_block_request(srv, sess, req)
    block = 0.08
    visible = [k for k in keys if k[0] * block + block - 0.2 >= -block]  # the stand-in frustum, margin = block
    got = [k for k, _ in sess.sent[0]]
    n_vis = min(40, len(visible))
    assert all(k in visible for k in got[: n_vis - 1])  # visible keys first (one of them was deleted)
    assert len(got) == 40 - 1 and (5, 1, 0) not in got
    assert all(raw == bytes([k[0] & 0xFF, k[1]]) for k, raw in sess.sent[0])
    assert sess.blocks_sent == len(got) and stream.size() == len(keys) - 40
