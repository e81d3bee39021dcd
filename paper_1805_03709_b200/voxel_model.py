"""TSDF block layout (voxel_model.py:23-72 of the reference) and the device
TSDF pool.

The pool stores each block as one 6,144-byte row in exactly the wire layout
(``TsdfBlock.to_bytes``): 512 voxels x {f32 tsdf, f32 weight, u8 rgb[3],
u8 pad}, x-fastest flat index x + 8y + 64z.  Keeping the wire layout on the
device makes ingest a plain copy and lets the encoder stage a whole block
with one TMA bulk copy.
"""

from __future__ import annotations

import numpy as np

BLOCK_EDGE = 8
BLOCK_VOXELS = BLOCK_EDGE ** 3

TSDF_VOXEL_DTYPE = np.dtype([("tsdf", "<f4"), ("weight", "<f4"), ("color", "u1", 3), ("pad", "u1")])
assert TSDF_VOXEL_DTYPE.itemsize == 12
TSDF_BLOCK_BYTES = BLOCK_VOXELS * TSDF_VOXEL_DTYPE.itemsize  # 6144

_idx = np.arange(BLOCK_VOXELS)
LOCAL_COORDS = np.stack([_idx % BLOCK_EDGE, (_idx // BLOCK_EDGE) % BLOCK_EDGE, _idx // (BLOCK_EDGE ** 2)],
                        axis=1).astype(np.int64)
del _idx


class TsdfBlock:
    """One 8x8x8 chunk of TSDF voxels (voxel_model.py:42-72), host container."""

    __slots__ = ("key", "tsdf", "weight", "color", "updated", "visible")

    def __init__(self, key) -> None:
        self.key = key
        self.tsdf = np.zeros(BLOCK_VOXELS, dtype=np.float32)
        self.weight = np.zeros(BLOCK_VOXELS, dtype=np.float32)
        self.color = np.zeros((BLOCK_VOXELS, 3), dtype=np.uint8)
        self.updated = False
        self.visible = False

    def to_bytes(self) -> bytes:
        return block_row(self).tobytes()

    @classmethod
    def from_bytes(cls, key, raw: bytes) -> "TsdfBlock":
        if len(raw) != TSDF_BLOCK_BYTES:
            raise ValueError(f"TSDF block payload must be {TSDF_BLOCK_BYTES} bytes")
        rec = np.frombuffer(raw, dtype=TSDF_VOXEL_DTYPE)
        blk = cls(key)
        blk.tsdf = rec["tsdf"].astype(np.float32)
        blk.weight = rec["weight"].astype(np.float32)
        blk.color = rec["color"].copy()
        blk.updated = True
        return blk


def block_row(blk) -> np.ndarray:
    """Any object with .tsdf/.weight/.color (e.g. a reference TsdfBlock) ->
    its 6,144-byte wire row as uint8."""
    rec = np.zeros(BLOCK_VOXELS, dtype=TSDF_VOXEL_DTYPE)
    rec["tsdf"] = blk.tsdf
    rec["weight"] = blk.weight
    rec["color"] = blk.color
    return rec.view(np.uint8)


def rows_from_soa(tsdf: np.ndarray, weight: np.ndarray, color: np.ndarray) -> np.ndarray:
    """SoA arrays [P,512], [P,512], [P,512,3] -> wire rows uint8[P,6144]."""
    P = tsdf.shape[0]
    rec = np.zeros((P, BLOCK_VOXELS), dtype=TSDF_VOXEL_DTYPE)
    rec["tsdf"] = tsdf
    rec["weight"] = weight
    rec["color"] = color
    return np.ascontiguousarray(rec.view(np.uint8).reshape(P, TSDF_BLOCK_BYTES))


# --------------------------------------------------------------------------
# RC-side voxel hashing on the GPU (voxel_model.py:105-299 of the reference)

import ctypes as _ct
import math as _math

_BOUNDARY_EPS = 1e-6  # voxel_model.py:102


class _RcParams(_ct.Structure):
    """Mirror of RcParams in csrc/fusion.cu (size checked at first use)."""

    _fields_ = [("R", _ct.c_double * 9), ("t", _ct.c_double * 3), ("R32", _ct.c_float * 9), ("t32", _ct.c_float * 3),
                ("fx", _ct.c_double), ("fy", _ct.c_double), ("cx", _ct.c_double), ("cy", _ct.c_double),
                ("width", _ct.c_int32), ("height", _ct.c_int32), ("voxel", _ct.c_double), ("mu", _ct.c_double),
                ("max_weight", _ct.c_double), ("block", _ct.c_double), ("tol", _ct.c_double),
                ("one_minus_tol", _ct.c_double), ("reach", _ct.c_double), ("stride", _ct.c_int32),
                ("steps", _ct.c_int32), ("ts", _ct.c_double * 64), ("planes", _ct.c_double * 24),
                ("margin", _ct.c_double)]


def _pose_arrays(pose):
    """Reference Pose (rotation, translation) or a (R, t) pair -> float64 arrays."""
    if hasattr(pose, "rotation"):
        return np.asarray(pose.rotation, np.float64), np.asarray(pose.translation, np.float64)
    R, t = pose
    return np.asarray(R, np.float64), np.asarray(t, np.float64)


def frustum_planes(R, t, intr, near: float, far: float) -> np.ndarray:
    """Frustum._build_planes (geometry.py:121-147), same numpy operations:
    (6,4) rows (nx, ny, nz, d), inward normals."""
    corners = np.array([
        [(0 - intr.cx) / intr.fx, (0 - intr.cy) / intr.fy, 1.0],
        [(intr.width - intr.cx) / intr.fx, (0 - intr.cy) / intr.fy, 1.0],
        [(intr.width - intr.cx) / intr.fx, (intr.height - intr.cy) / intr.fy, 1.0],
        [(0 - intr.cx) / intr.fx, (intr.height - intr.cy) / intr.fy, 1.0],
    ])
    rays = corners @ R.T
    origin = t
    fwd = R[:, 2]
    planes = []

    def plane(normal, point):
        normal = normal / np.linalg.norm(normal)
        planes.append([*normal, -float(normal @ point)])

    plane(fwd, origin + near * fwd)
    plane(-fwd, origin + far * fwd)
    for a, b in ((0, 1), (1, 2), (2, 3), (3, 0)):
        plane(np.cross(rays[a], rays[b]), origin)
    return np.asarray(planes, dtype=np.float64)


class GpuVoxelModel:
    """Device-resident sparse TSDF model with the reference VoxelModel's
    allocation and fusion (voxel_model.py:144-299).  Blocks live in a GPU
    hash map whose positions index a wire-layout TSDF pool (the map's
    parallel payload array), so the fused blocks feed the MC encoder and the
    server ingest directly.

    cfg: a FusionConfig-like object (voxel_size, truncation, max_weight,
    alloc_stride); intrinsics: CameraIntrinsics-like (fx, fy, cx, cy, width,
    height); pose: a Pose-like (rotation, translation) or an (R, t) pair.
    """

    def __init__(self, cfg, bucket_count: int = 1 << 17, excess_capacity: int = 1 << 17, device=None) -> None:
        from . import _lib
        from .concurrent_hash import BlockHashSet

        torch = _lib.require_cuda()
        self._torch = torch
        self._lib = _lib
        self.cfg = cfg
        self.blocks = BlockHashSet(bucket_count, excess_capacity, device=device)
        self.device = self.blocks.device
        self.pool = torch.zeros((self.blocks.capacity, TSDF_BLOCK_BYTES), dtype=torch.uint8, device=self.device)
        if _lib.load().vs_rc_params_bytes() != _ct.sizeof(_RcParams):
            raise RuntimeError("RcParams layout mismatch between Python and libvsb200")

    @property
    def block_size(self) -> float:
        return BLOCK_EDGE * self.cfg.voxel_size

    def _params(self, pose, intr, planes: bool) -> _RcParams:
        cfg = self.cfg
        R, t = _pose_arrays(pose)
        p = _RcParams()
        p.R[:] = R.reshape(-1).tolist()
        p.t[:] = t.tolist()
        p.R32[:] = R.astype(np.float32).reshape(-1).tolist()
        p.t32[:] = t.astype(np.float32).tolist()
        p.fx, p.fy, p.cx, p.cy = float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy)
        p.width, p.height = int(intr.width), int(intr.height)
        p.voxel, p.mu, p.max_weight = float(cfg.voxel_size), float(cfg.truncation), float(cfg.max_weight)
        p.block = BLOCK_EDGE * cfg.voxel_size
        p.tol = _BOUNDARY_EPS / p.block
        p.one_minus_tol = 1.0 - p.tol
        p.reach = cfg.truncation + p.block * np.sqrt(3.0)
        p.stride = int(getattr(cfg, "alloc_stride", 1))
        steps = int(np.ceil(2 * cfg.truncation / cfg.voxel_size)) + 1
        if steps > 64:
            raise ValueError("truncation / voxel_size too large for the device step table (max 64 steps)")
        p.steps = steps
        p.ts[:steps] = np.linspace(0.0, 1.0, steps).tolist()
        if planes:
            # sensor_frustum(pose, intr, margin=block_size), near 0.05, far 20 (voxel_model.py:212, 303-313)
            p.planes[:] = frustum_planes(R, t, intr, 0.05, 20.0).reshape(-1).tolist()
            p.margin = p.block
        return p

    def _img(self, a, dtype):
        t = self._torch.as_tensor(np.ascontiguousarray(a)) if not isinstance(a, self._torch.Tensor) else a
        return t.to(self.device, dtype).contiguous()

    def allocate_blocks(self, depth, pose, intrinsics) -> list:
        """Ensure blocks along every valid ray segment [d-mu, d+mu]; returns the
        newly created keys in sorted order, like the reference."""
        new = self.allocate_blocks_tensor(depth, pose, intrinsics, sort=True)
        return [tuple(r) for r in new.cpu().tolist()]

    def allocate_blocks_tensor(self, depth, pose, intrinsics, sort: bool = False):
        """Device fast path of allocate_blocks -> int32[m,3] created keys."""
        torch = self._torch
        lib = self._lib
        d = self._img(depth, torch.float32)
        P = self._params(pose, intrinsics, planes=False)
        s = self.blocks._stream()
        # candidate buffer sized by the largest count seen so far (one pass per frame)
        cap = max(getattr(self, "_cand_cap", 0), 1 << 16, 2 * d.numel())
        n_dev = torch.zeros(1, dtype=torch.int64, device=self.device)
        while True:
            cand = torch.empty((cap, 3), dtype=torch.int32, device=self.device)
            lib.check(lib.load().vs_rc_candidates(lib.ptr(d), _ct.byref(P), lib.ptr(cand), cap, lib.ptr(n_dev),
                                                  _ct.c_void_p(s.cuda_stream)), "rc_candidates")
            n = int(n_dev.item())
            if n <= cap:
                break
            cap = n + n // 4
        self._cand_cap = cap
        cand = cand[:n]
        self.blocks._done(s)
        created, pos = self.blocks.insert_many_exact(cand)
        s = self.blocks._stream()
        lib.check(lib.load().vs_rc_zero_rows(lib.ptr(pos), lib.ptr(created), n, lib.ptr(self.pool),
                                             _ct.c_void_p(s.cuda_stream)), "rc_zero_rows")
        self.blocks._done(s)
        new = cand[created.bool()]
        if not sort or new.shape[0] == 0:
            return new
        k = new.to(torch.int64)
        off = 1 << 20
        enc = ((k[:, 0] + off) << 42) | ((k[:, 1] + off) << 21) | (k[:, 2] + off)
        return new[torch.argsort(enc)]

    def fuse_frame_async(self, depth, color, pose, intrinsics):
        """allocate_blocks + integrate_frame of one frame with NO host
        synchronisation (pipelines and the bench): candidates into a buffer
        sized by the largest count seen so far, a device-count-bounded insert
        (vs_table_insert_bounded), fresh rows zeroed, integration over the
        map.  Returns (touched_keys_buffer, touched_n_dev).  The exact
        per-frame failure semantics of allocate_blocks are not kept here:
        call check_async() (synchronising) after a run of frames -- it raises
        if a candidate buffer overflowed or the excess list ran dry."""
        torch = self._torch
        lib = self._lib
        L = lib.load()
        d = self._img(depth, torch.float32)
        c = self._img(color, torch.uint8)
        cap = max(getattr(self, "_cand_cap", 0), 1 << 16, 2 * d.numel())
        if getattr(self, "_async", None) is None or self._async["cap"] < cap:
            self._async = {"cap": cap,
                           "cand": torch.empty((cap, 3), dtype=torch.int32, device=self.device),
                           "created": torch.empty(cap, dtype=torch.uint8, device=self.device),
                           "pos": torch.empty(cap, dtype=torch.int32, device=self.device),
                           "n": torch.zeros(1, dtype=torch.int64, device=self.device),
                           "n_max": torch.zeros(1, dtype=torch.int64, device=self.device)}
        if getattr(self, "_touched_buf", None) is None:
            self._touched_buf = torch.empty((self.blocks.capacity, 3), dtype=torch.int32, device=self.device)
            self._touched_n = torch.zeros(1, dtype=torch.int64, device=self.device)
        a = self._async
        s = self.blocks._stream()
        st = _ct.c_void_p(s.cuda_stream)
        P = self._params(pose, intrinsics, planes=False)
        lib.check(L.vs_rc_candidates(lib.ptr(d), _ct.byref(P), lib.ptr(a["cand"]), a["cap"], lib.ptr(a["n"]), st),
                  "rc_candidates")
        torch.maximum(a["n_max"], a["n"], out=a["n_max"])  # overflow check deferred to check_async
        lib.check(L.vs_table_insert_bounded(self.blocks.handle, lib.ptr(a["cand"]), a["cap"], lib.ptr(a["n"]),
                                            lib.ptr(a["created"]), lib.ptr(a["pos"]), st), "insert_bounded")
        lib.check(L.vs_rc_zero_rows(lib.ptr(a["pos"]), lib.ptr(a["created"]), a["cap"], lib.ptr(self.pool), st),
                  "rc_zero_rows")
        P = self._params(pose, intrinsics, planes=True)
        lib.check(L.vs_rc_integrate_table(self.blocks._h, lib.ptr(d), lib.ptr(c), _ct.byref(P), lib.ptr(self.pool),
                                          lib.ptr(self._touched_buf), lib.ptr(self._touched_n), st), "rc_integrate")
        self.blocks._done(s)
        return self._touched_buf, self._touched_n

    def check_async(self) -> None:
        """Synchronise and verify a run of fuse_frame_async frames."""
        a = getattr(self, "_async", None)
        if a is not None and int(a["n_max"].item()) > a["cap"]:
            raise RuntimeError(f"candidate buffer overflow ({int(a['n_max'].item())} > {a['cap']}): "
                               "run a synchronous frame first to size it")
        self.blocks.check_capacity()

    def integrate_frame(self, depth, color, pose, intrinsics) -> list:
        """Fuse one registered RGB-D frame into all allocated in-view blocks;
        returns the keys that received at least one voxel update."""
        return [tuple(r) for r in self.integrate_frame_tensor(depth, color, pose, intrinsics).cpu().tolist()]

    def integrate_frame_tensor(self, depth, color, pose, intrinsics):
        """Device fast path of integrate_frame -> int32[m,3] touched keys
        (ascending pool row).  Walks the map's entry slots directly (pool
        row = slot), so no snapshot is taken; one host sync for the count."""
        torch = self._torch
        lib = self._lib
        d = self._img(depth, torch.float32)
        c = self._img(color, torch.uint8)
        P = self._params(pose, intrinsics, planes=True)
        if getattr(self, "_touched_buf", None) is None:
            self._touched_buf = torch.empty((self.blocks.capacity, 3), dtype=torch.int32, device=self.device)
            self._touched_n = torch.zeros(1, dtype=torch.int64, device=self.device)
        s = self.blocks._stream()
        lib.check(lib.load().vs_rc_integrate_table(self.blocks._h, lib.ptr(d), lib.ptr(c), _ct.byref(P),
                                                   lib.ptr(self.pool), lib.ptr(self._touched_buf),
                                                   lib.ptr(self._touched_n), _ct.c_void_p(s.cuda_stream)),
                  "rc_integrate")
        n = int(self._touched_n.item())
        out = self._touched_buf[:n].clone()
        self.blocks._done(s)
        return out

    def keys(self) -> list:
        return self.blocks.snapshot_keys()

    def rows(self, keys):
        """Wire rows (uint8[N,6144], device) of the given keys (zeros if absent)."""
        found, pos = self.blocks.find_keys(keys)
        out = self.pool[pos.clamp(min=0).long()]
        out[~found.bool()] = 0
        return out

    def get_block(self, key):
        found, pos = self.blocks.find_keys([key])
        if not bool(found[0].item()):
            return None
        raw = self.pool[int(pos[0].item())].cpu().numpy().tobytes()
        return TsdfBlock.from_bytes(key, raw)
