"""CPU test of the drop-in installer against a stand-in package with the
reference's module/attribute layout (the real reference is not available on
the GPU box, and constructing tables needs a GPU, so only the rebinding is
checked here; INTEGRATION.md shows the real use)."""

from __future__ import annotations

import sys
import types


def _fake_package(name):
    pkg = types.ModuleType(name)
    pkg.__path__ = []
    sys.modules[name] = pkg
    mods = {}
    for m in ("concurrent_hash", "server", "voxel_model", "exploration", "mc_encoding", "reconstruction"):
        mod = types.ModuleType(f"{name}.{m}")
        sys.modules[f"{name}.{m}"] = mod
        setattr(pkg, m, mod)
        mods[m] = mod
    for m in ("concurrent_hash", "server", "voxel_model", "exploration"):
        mods[m].BlockHashMap = object
    mods["concurrent_hash"].BlockHashSet = object
    mods["server"].BlockHashSet = object
    mods["server"].StreamSet = object
    mods["reconstruction"].StreamSet = object
    mods["server"].recompute_mc_block = None

    class Server:
        def on_tsdf_batch(self, batch):
            return "reference"

        def on_block_request(self, sess, req):
            return "reference"

        def on_reset_blocks(self, keys):
            return "reference"

    mods["server"].Server = Server
    pkg.BlockHashSet = object
    pkg.BlockHashMap = object
    pkg.recompute_mc_block = None
    return pkg, mods


def test_install_rebinds_hot_path_names_and_uninstall_restores():
    from paper_1805_03709_b200 import concurrent_hash as gch
    from paper_1805_03709_b200 import mc_encoding as gmc
    from paper_1805_03709_b200 import server as gsrv
    from paper_1805_03709_b200 import shim

    pkg, mods = _fake_package("fakevs_ref")
    original = mods["server"].Server.on_tsdf_batch
    shim.install("fakevs_ref")
    try:
        assert mods["concurrent_hash"].BlockHashSet is gch.BlockHashSet
        assert mods["concurrent_hash"].BlockHashMap is gch.BlockHashMap
        assert mods["server"].BlockHashSet is gch.BlockHashSet
        assert mods["server"].StreamSet is gsrv.StreamSet
        assert mods["reconstruction"].StreamSet is gsrv.StreamSet
        assert mods["voxel_model"].BlockHashMap is gch.BlockHashMap
        assert mods["exploration"].BlockHashMap is gch.BlockHashMap
        assert mods["server"].recompute_mc_block is gmc.recompute_mc_block
        assert pkg.BlockHashSet is gch.BlockHashSet
        assert mods["server"].Server.on_tsdf_batch is shim._on_tsdf_batch
        assert mods["server"].Server.on_block_request is shim._on_block_request
        assert mods["server"].Server.on_reset_blocks is shim._on_reset_blocks
    finally:
        shim.uninstall()
    assert mods["concurrent_hash"].BlockHashSet is object
    assert mods["server"].StreamSet is object
    assert mods["server"].Server.on_tsdf_batch is original
    for k in [k for k in sys.modules if k.startswith("fakevs_ref")]:
        del sys.modules[k]


def test_block_request_batches_the_map_lookups():
    """shim._on_block_request (server.py:334-363): strategy dispatch, ONE
    get_many for the whole request, keys deleted meanwhile dropped, the
    request counted, and the keys given back when the send fails."""
    import enum

    from paper_1805_03709_b200 import shim

    class Strategy(enum.IntEnum):
        GENERATION_ORDER = 0
        VISIBLE_FIRST = 1
        RANDOM = 2

    class McBatch:
        def __init__(self, blocks):
            self.blocks = blocks

    mod = types.ModuleType("fake_block_server")
    mod.wire = types.SimpleNamespace(Strategy=Strategy, McBatch=McBatch)
    sys.modules[mod.__name__] = mod

    class Stream:  # a host stream set (the device path is tested on the GPU)
        def __init__(self, keys):
            self.keys = list(keys)
            self.back = []

        def extract_random(self, n):
            out, self.keys = self.keys[:n], self.keys[n:]
            return out

        def extract_ordered(self, n):
            return self.extract_random(n)

        def extract_matching(self, n, pred):
            out = [k for k in self.keys if pred(k)][:n]
            self.keys = [k for k in self.keys if k not in out]
            return out

        def insert_many(self, keys):
            self.back.extend(keys)

    class Map:
        def __init__(self):
            self.calls = 0

        def get_many(self, keys):
            self.calls += 1
            return [None if k[0] == 3 else bytes([k[0]]) for k in keys]

    class Sess:
        def __init__(self, stream, ok=True):
            self.stream, self.ok = stream, ok
            self.request_count = self.blocks_sent = 0
            self.sent = []

        def send(self, msg, codec):
            self.sent.append(msg.blocks)
            return self.ok

    Server = type("Server", (), {"__module__": mod.__name__})
    srv = Server()
    srv.cfg = types.SimpleNamespace(max_request_blocks=4, codec=None, voxel_size=0.01)
    srv.mc_map = Map()
    srv._delivery_lock = __import__("threading").Lock()
    srv._visibility_predicate = lambda req: (lambda k: k[1] == 0)
    keys = [(i, i % 2, 0) for i in range(10)]
    for strategy, want in ((Strategy.RANDOM, [0, 1, 2, 3]), (Strategy.GENERATION_ORDER, [0, 1, 2, 3]),
                           (Strategy.VISIBLE_FIRST, [0, 2, 4, 6])):  # max_request_blocks = 4
        sess = Sess(Stream(keys))
        req = types.SimpleNamespace(max_blocks=10, strategy=strategy)
        shim._on_block_request(srv, sess, req)
        got = [k[0] for k, _ in sess.sent[0]]
        assert got == [k for k in want if k != 3], (strategy, got)
        assert sess.request_count == 1 and sess.blocks_sent == len(got)
    assert srv.mc_map.calls == 3  # one lookup per request, not one per key
    sess = Sess(Stream(keys), ok=False)
    shim._on_block_request(srv, sess, types.SimpleNamespace(max_blocks=2, strategy=Strategy.RANDOM))
    assert sess.stream.back == [(0, 0, 0), (1, 1, 0)] and sess.blocks_sent == 0


def test_reset_blocks_batched_removes():
    """shim._on_reset_blocks (server.py:425-436): keys leave both maps (one
    remove_many each) and every client's set, every client gets DeleteBlocks."""
    from paper_1805_03709_b200 import shim

    class DeleteBlocks:
        def __init__(self, keys):
            self.keys = keys

    mod = types.ModuleType("fake_reset_server")
    mod.wire = types.SimpleNamespace(DeleteBlocks=DeleteBlocks)
    sys.modules[mod.__name__] = mod

    class Map:
        def __init__(self, keys):
            self.keys, self.calls = set(keys), 0

        def remove_many(self, keys):
            self.calls += 1
            n = len(self.keys & set(keys))
            self.keys -= set(keys)
            return n

    class HostSet:
        def __init__(self, keys):
            self.keys = set(keys)

        def remove(self, key):
            had = key in self.keys
            self.keys.discard(key)
            return had

    class Ec:
        def __init__(self, keys):
            self.stream = HostSet(keys)
            self.sent = []

        def send(self, msg, codec):
            self.sent.append(msg.keys)

    allk = [(i, 0, 0) for i in range(10)]
    Server = type("Server", (), {"__module__": mod.__name__})
    srv = Server()
    srv.cfg = types.SimpleNamespace(codec=None)
    srv.tsdf_map, srv.mc_map = Map(allk), Map(allk)
    ecs = [Ec(allk), Ec(allk[:5])]
    srv._exploration_sessions = lambda: ecs
    srv._delivery_lock = __import__("threading").Lock()
    gone = allk[3:7]
    shim._on_reset_blocks(srv, gone)
    for m in (srv.tsdf_map, srv.mc_map):
        assert m.keys == set(allk) - set(gone) and m.calls == 1
    assert ecs[0].stream.keys == set(allk) - set(gone) and ecs[1].stream.keys == set(allk[:3])
    assert all(ec.sent == [gone] for ec in ecs)
    shim._on_reset_blocks(srv, [])
    assert all(len(ec.sent) == 1 for ec in ecs)


def test_install_can_keep_client_side_host_maps():
    from paper_1805_03709_b200 import concurrent_hash as gch
    from paper_1805_03709_b200 import shim

    pkg, mods = _fake_package("fakevs_ref2")
    shim.install("fakevs_ref2", client_maps=False)
    try:
        assert mods["server"].BlockHashMap is gch.BlockHashMap
        assert mods["voxel_model"].BlockHashMap is object and mods["exploration"].BlockHashMap is object
    finally:
        shim.uninstall()
