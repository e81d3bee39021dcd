"""RC-side voxel hashing on the GPU (allocate_blocks + integrate_frame,
voxel_model.py:165-299) replayed on the reference's own sphere sequence
(tests/golden/fusion_sphere.npz, recorded from the reference): per-frame
created keys and touched keys, the final TSDF blocks bit for bit, and the
MC encoding of the fused model reproducing manifest.json's model_sha256."""

from __future__ import annotations

import hashlib
import json
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _inputs(golden):
    d = np.load(golden / "fusion_sphere.npz")
    fx, fy, cx, cy, w, h = d["intr"].tolist()
    intr = types.SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))
    voxel, mu, maxw, stride = d["cfg"].tolist()
    cfg = types.SimpleNamespace(voxel_size=voxel, truncation=mu, max_weight=maxw, alloc_stride=int(stride))
    return d, intr, cfg


def test_sphere_fusion_bit_exact_and_model_digest(dev, golden):
    from paper_1805_03709_b200 import encode_keys
    from paper_1805_03709_b200.voxel_model import GpuVoxelModel, rows_from_soa

    d, intr, cfg = _inputs(golden)
    model = GpuVoxelModel(cfg, bucket_count=1 << 13, excess_capacity=1 << 13)
    c_off = np.concatenate([[0], np.cumsum(d["created_counts"])])
    t_off = np.concatenate([[0], np.cumsum(d["touched_counts"])])
    for f in range(d["depth"].shape[0]):
        R, t = d["pose"][f][:9].reshape(3, 3), d["pose"][f][9:]
        new = model.allocate_blocks(d["depth"][f], (R, t), intr)
        assert new == [tuple(k) for k in d["created"][c_off[f]:c_off[f + 1]].tolist()], f  # sorted, exact
        touched = model.integrate_frame(d["depth"][f], d["color"][f], (R, t), intr)
        assert set(touched) == {tuple(k) for k in d["touched"][t_off[f]:t_off[f + 1]].tolist()}, f
    s = np.load(golden / "mc_sphere.npz")
    keys = s["keys"]
    assert sorted(model.keys()) == [tuple(k) for k in keys.tolist()]
    got = model.rows(keys).cpu().numpy()
    want = rows_from_soa(s["tsdf"], s["weight"], s["color"])
    assert np.array_equal(got, want)  # every fused voxel (tsdf, weight, colour) bit for bit
    mc, _, _ = encode_keys(model.blocks, model.pool, keys)
    meta = json.loads((golden / "mc_sphere.json").read_text())
    assert hashlib.sha256(mc.cpu().numpy().tobytes()).hexdigest() == meta["model_sha256"]


def test_sync_free_fusion_path_reproduces_the_reference_model(dev, golden):
    """fuse_frame_async (no host sync per frame: device-bounded insert,
    zeroed rows, integration over the map) on the reference's sphere
    sequence: the same keys and the same voxels bit for bit, and the MC
    digest of manifest.json."""
    from paper_1805_03709_b200 import encode_keys
    from paper_1805_03709_b200.voxel_model import GpuVoxelModel, rows_from_soa

    d, intr, cfg = _inputs(golden)
    model = GpuVoxelModel(cfg, bucket_count=1 << 13, excess_capacity=1 << 13)
    for f in range(d["depth"].shape[0]):
        R, t = d["pose"][f][:9].reshape(3, 3), d["pose"][f][9:]
        model.fuse_frame_async(d["depth"][f], d["color"][f], (R, t), intr)
    model.check_async()
    s = np.load(golden / "mc_sphere.npz")
    keys = s["keys"]
    assert sorted(model.keys()) == [tuple(k) for k in keys.tolist()]
    assert np.array_equal(model.rows(keys).cpu().numpy(), rows_from_soa(s["tsdf"], s["weight"], s["color"]))
    mc, _, _ = encode_keys(model.blocks, model.pool, keys)
    meta = json.loads((golden / "mc_sphere.json").read_text())
    assert hashlib.sha256(mc.cpu().numpy().tobytes()).hexdigest() == meta["model_sha256"]


def test_reallocation_is_idempotent_and_get_block(dev, golden):
    from paper_1805_03709_b200.voxel_model import GpuVoxelModel

    d, intr, cfg = _inputs(golden)
    model = GpuVoxelModel(cfg, bucket_count=1 << 13, excess_capacity=1 << 13)
    R, t = d["pose"][0][:9].reshape(3, 3), d["pose"][0][9:]
    first = model.allocate_blocks(d["depth"][0], (R, t), intr)
    assert len(first) == d["created_counts"][0]
    assert model.allocate_blocks(d["depth"][0], (R, t), intr) == []  # re-running creates nothing
    blk = model.get_block(first[0])
    assert blk is not None and not blk.weight.any()  # fresh TsdfBlock(): zeros
    assert model.get_block((10 ** 6, 0, 0)) is None


def test_room_frames_gpu_vs_oracle(dev):
    """Synthetic room RGB-D frames (analytic ray-box depth): GPU fusion ==
    the numpy restatement, created keys / touched keys / every voxel."""
    from oracle.fusion_oracle import OracleVoxelModel
    from paper_1805_03709_b200 import workloads
    from paper_1805_03709_b200.voxel_model import GpuVoxelModel, rows_from_soa

    depth, color, Rs, ts, (fx, fy, cx, cy, w, h) = workloads.room_frames(4, 160, 120)
    intr = types.SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)
    cfg = types.SimpleNamespace(voxel_size=0.02, truncation=0.08, max_weight=128.0, alloc_stride=1)
    gpu = GpuVoxelModel(cfg, bucket_count=1 << 15, excess_capacity=1 << 15)
    ref = OracleVoxelModel(0.02, 0.08)
    for f in range(4):
        a = gpu.allocate_blocks(depth[f], (Rs[f], ts[f]), intr)
        b = ref.allocate(depth[f], Rs[f], ts[f], float(fx), float(fy), float(cx), float(cy))
        assert a == b, f
        ta = gpu.integrate_frame(depth[f], color[f], (Rs[f], ts[f]), intr)
        tb = ref.integrate(depth[f], color[f], Rs[f], ts[f], float(fx), float(fy), float(cx), float(cy))
        assert set(ta) == set(tb), f
    keys = sorted(ref.blocks)
    assert sorted(gpu.keys()) == keys
    want = rows_from_soa(np.stack([ref.blocks[k][0] for k in keys]), np.stack([ref.blocks[k][1] for k in keys]),
                         np.stack([ref.blocks[k][2] for k in keys]))
    assert np.array_equal(gpu.rows(np.asarray(keys, np.int32)).cpu().numpy(), want)


def test_integrate_keys_abi_matches_table_walk(dev):
    """vs_rc_integrate (explicit keys + pool rows, e.g. a snapshot) and
    vs_rc_integrate_table (walks the map's slots) give the same rows and
    flag the same blocks; the table walk returns ascending slots."""
    import ctypes

    import torch

    from paper_1805_03709_b200 import _lib, workloads
    from paper_1805_03709_b200.voxel_model import GpuVoxelModel

    depth, color, Rs, ts, (fx, fy, cx, cy, w, h) = workloads.room_frames(3, 160, 120)
    intr = types.SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)
    cfg = types.SimpleNamespace(voxel_size=0.02, truncation=0.08, max_weight=128.0, alloc_stride=1)
    a = GpuVoxelModel(cfg, bucket_count=1 << 15, excess_capacity=1 << 15)
    b = GpuVoxelModel(cfg, bucket_count=1 << 15, excess_capacity=1 << 15)
    lib = _lib.load()
    for f in range(3):
        a.allocate_blocks(depth[f], (Rs[f], ts[f]), intr)
        b.allocate_blocks(depth[f], (Rs[f], ts[f]), intr)
        ta = a.integrate_frame_tensor(torch.from_numpy(depth[f]).to(dev), torch.from_numpy(color[f]).to(dev),
                                      (Rs[f], ts[f]), intr)
        keys, pos = b.blocks.snapshot_tensor()
        touched = torch.empty(keys.shape[0], dtype=torch.uint8, device=dev)
        P = b._params((Rs[f], ts[f]), intr, planes=True)
        d = torch.from_numpy(depth[f]).to(dev)
        c = torch.from_numpy(color[f]).contiguous().to(dev)
        _lib.check(lib.vs_rc_integrate(_lib.ptr(keys), _lib.ptr(pos), keys.shape[0], _lib.ptr(d), _lib.ptr(c),
                                       ctypes.byref(P), _lib.ptr(b.pool), _lib.ptr(touched),
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "rc_integrate")
        tb = keys[touched.bool()]
        assert ta.shape[0] > 0
        slot = a.blocks.find_keys(ta)[1]
        assert bool((slot[1:] > slot[:-1]).all())
        # same set (slot assignment of the two maps may differ)
        assert sorted(map(tuple, ta.tolist())) == sorted(map(tuple, tb.tolist())), f
    keys, _ = a.blocks.snapshot_tensor()
    assert torch.equal(a.rows(keys), b.rows(keys))
