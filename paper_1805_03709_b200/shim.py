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
  voxelstream.server.Server.on_block_request                 -> batched:
        one map lookup for the whole request instead of one per key, and
        the VISIBLE_FIRST frustum test on the device (server.py:334-387)
  voxelstream.server.Server.on_reset_blocks                  -> batched:
        one remove launch per map and one for every client set instead of
        K x (2 + clients) per-key removes (server.py:425-436)

Modules bind names at import time (server.py:25, voxel_model.py:20,
exploration.py:24), so both the defining module and the importers are
patched.  ``uninstall()`` restores the originals.
"""

from __future__ import annotations

import sys
from typing import Any
from . import server as _gserver

_saved: list[tuple[Any, str, Any]] = []


def _set(obj, name: str, value) -> None:
    if hasattr(obj, name):
        _saved.append((obj, name, getattr(obj, name)))
        setattr(obj, name, value)


def install(package: str = "voxelstream", batched_server: bool = True, client_maps: bool = True) -> None:
    """Patch the (already importable) reference package in place.

    client_maps=False keeps the reference's host maps in ``voxel_model`` and
    ``exploration``: their per-key loops (VoxelModel.allocate_blocks /
    integrate_frame, ExplorationClient) would pay one GPU round trip per key
    (INTEGRATION.md); reconstruction clients get the batched
    ``voxel_model.GpuVoxelModel`` instead."""
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
    client_side = {mods.get("voxel_model"), mods.get("exploration")} - {None}
    for mod in list(mods.values()) + [top]:
        if not client_maps and mod in client_side:
            continue
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
            _set(srv.Server, "on_block_request", _on_block_request)
            _set(srv.Server, "on_reset_blocks", _on_reset_blocks)
    _set(top, "recompute_mc_block", gmc.recompute_mc_block)


def uninstall() -> None:
    while _saved:
        obj, name, value = _saved.pop()
        setattr(obj, name, value)


@_gserver._locked
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


def _frustum_args(self, req, srv):
    """The frustum _visibility_predicate builds (server.py:365-375), as the
    (planes, margin, block size) the device predicate takes."""
    voxel = self.cfg.voxel_size or 0.005
    block_size = srv.BLOCK_EDGE * voxel
    fx, fy, cx, cy, near, far = req.intrinsics
    pose = srv.Pose.from_floats(req.pose)
    intr = srv.CameraIntrinsics(fx=fx, fy=fy, cx=cx, cy=cy, width=int(2 * cx) or 640, height=int(2 * cy) or 480)
    frustum = srv.Frustum(pose, intr, near=max(near, 1e-3), far=far, margin=block_size)
    return frustum._planes, frustum.margin, block_size


@_gserver._locked
def _on_block_request(self, sess, req) -> None:
    """server.py:334-363 with the same strategies and effects, but ONE
    batched map lookup for the requested keys (mc_map.get per key is one GPU
    round trip each), and for VISIBLE_FIRST on a GPU stream set the frustum
    test on the device (extract_visible_first: decisions bit-identical to
    _visibility_predicate, same random top-up)."""
    from . import server as gsrv

    if sess.stream is None:
        return
    srv = sys.modules[type(self).__module__]
    wire = srv.wire
    n = min(req.max_blocks, self.cfg.max_request_blocks)
    stream = sess.stream
    strategy = req.strategy
    if strategy == wire.Strategy.VISIBLE_FIRST:
        if isinstance(stream, gsrv.StreamSet):
            planes, margin, block = _frustum_args(self, req, srv)
            keys = stream.extract_visible_first(n, planes, margin, block)
        else:
            keys = stream.extract_matching(n, self._visibility_predicate(req))
            if len(keys) < n:  # top up so requests stay full-sized
                keys.extend(stream.extract_random(n - len(keys)))
    elif strategy == wire.Strategy.GENERATION_ORDER:
        keys = stream.extract_ordered(n)
    else:
        keys = stream.extract_random(n)
    sess.request_count += 1
    with self._delivery_lock:
        get_many = getattr(self.mc_map, "get_many", None)
        raws = get_many(keys) if get_many is not None else [self.mc_map.get(k) for k in keys]
        blocks = [(k, raw) for k, raw in zip(keys, raws) if raw is not None]  # deleted by a reset meanwhile
        ok = sess.send(wire.McBatch(blocks), self.cfg.codec)
    if ok:
        sess.blocks_sent += len(blocks)
    else:
        # connection died mid-delivery: nothing may be lost
        stream.insert_many(keys)


@_gserver._locked
def _on_reset_blocks(self, keys) -> None:
    """server.py:425-436 with the same effects (keys gone from both maps and
    every exploration client's set, DeleteBlocks sent to each client), the
    removes batched: one launch per map, one for all GPU client sets."""
    from . import server as gsrv

    if not keys:
        return
    srv = sys.modules[type(self).__module__]
    wire = srv.wire
    ecs = self._exploration_sessions()
    with self._delivery_lock:
        for m in (self.tsdf_map, self.mc_map):
            if hasattr(m, "remove_many"):
                m.remove_many(keys)
            else:
                for key in keys:
                    m.remove(key)
        gpu = [ec.stream for ec in ecs if isinstance(ec.stream, gsrv.StreamSet)]
        if gpu:
            gsrv.remove_everywhere(gpu, keys)
        for ec in ecs:
            if not isinstance(ec.stream, gsrv.StreamSet):
                for key in keys:
                    ec.stream.remove(key)
            ec.send(wire.DeleteBlocks(keys), self.cfg.codec)
