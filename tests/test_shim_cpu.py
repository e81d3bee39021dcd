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
    finally:
        shim.uninstall()
    assert mods["concurrent_hash"].BlockHashSet is object
    assert mods["server"].StreamSet is object
    assert mods["server"].Server.on_tsdf_batch is original
    for k in [k for k in sys.modules if k.startswith("fakevs_ref")]:
        del sys.modules[k]
