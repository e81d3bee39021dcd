"""Install the GPU path under the reference package ``voxelstream``.

``install()`` rebinds the hot-path names in the already-imported reference
modules, the maintainers' one-line integration:

  voxelstream.concurrent_hash.BlockHashSet / BlockHashMap   -> GPU tables
  voxelstream.server.BlockHashSet / BlockHashMap / StreamSet -> GPU versions
  voxelstream.voxel_model.BlockHashMap, voxelstream.exploration.BlockHashMap
  voxelstream.server.recompute_mc_block                      -> GPU encoder
  voxelstream.server.Server.on_tsdf_batch                    -> batched:
        one encode launch per TSDF batch and one fan-out launch for all
        exploration clients instead of per-block / per-key Python loops
        (server.py:299-315)

Modules bind names at import time (server.py:25, voxel_model.py:20,
exploration.py:24), so both the defining module and the importers are
patched.  ``uninstall()`` restores the originals.
"""

from __future__ import annotations

import sys
from typing import Any

_saved: list[tuple[Any, str, Any]] = []


def _set(obj, name: str, value) -> None:
    if hasattr(obj, name):
        _saved.append((obj, name, getattr(obj, name)))
        setattr(obj, name, value)


def install(package: str = "voxelstream", batched_server: bool = True) -> None:
    """Patch the (already importable) reference package in place."""
    import importlib

    from . import concurrent_hash as gch
    from . import mc_encoding as gmc
    from . import server as gsrv

    mods = {}
    for m in ("concurrent_hash", "server", "voxel_model", "exploration", "mc_encoding", "reconstruction"):
        try:
            mods[m] = importlib.import_module(f"{package}.{m}")
        except ImportError:
            continue
    top = sys.modules.get(package) or importlib.import_module(package)
    for mod in list(mods.values()) + [top]:
        _set(mod, "BlockHashSet", gch.BlockHashSet)
        _set(mod, "BlockHashMap", gch.BlockHashMap)
    srv = mods.get("server")
    if srv is not None:
        _set(srv, "StreamSet", gsrv.StreamSet)
        _set(srv, "recompute_mc_block", gmc.recompute_mc_block)
        rc = mods.get("reconstruction")
        if rc is not None:
            _set(rc, "StreamSet", gsrv.StreamSet)
        if batched_server and hasattr(srv, "Server"):
            _set(srv.Server, "on_tsdf_batch", _on_tsdf_batch)
    _set(top, "recompute_mc_block", gmc.recompute_mc_block)


def uninstall() -> None:
    while _saved:
        obj, name, value = _saved.pop()
        setattr(obj, name, value)


def _on_tsdf_batch(self, batch) -> None:
    """server.py:299-315 with one GPU encode + one fan-out launch per batch.

    Same observable effects as the reference: TSDF put per block (latest
    write wins), affected = ordered first-occurrence dedup, MC put per
    affected key, insert_many of the recomputed keys into every exploration
    client (FIFO in affected order).
    """
    from . import mc_encoding as gmc
    from . import server as gsrv
    from .mc_encoding import affected_mc_blocks

    srv = sys.modules[type(self).__module__]
    TsdfBlock = srv.TsdfBlock
    updated = []
    for key, raw in batch.blocks:
        self.tsdf_map.put(key, TsdfBlock.from_bytes(key, raw))
        updated.append(key)
    affected = list(dict.fromkeys(nb for key in updated for nb in affected_mc_blocks(key)))
    for mc in gmc.recompute_mc_blocks(affected, self.tsdf_map.get):
        self.mc_map.put(mc.key, mc.to_bytes())
    streams = [ec.stream for ec in self._exploration_sessions()]
    gpu = [s for s in streams if isinstance(s, gsrv.StreamSet)]
    if gpu:
        gsrv.fan_out(gpu, affected)
    for s in streams:
        if not isinstance(s, gsrv.StreamSet):
            s.insert_many(affected)
