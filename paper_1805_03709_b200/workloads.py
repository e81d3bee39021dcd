"""Seeded synthetic workloads of BASELINE.json's configs.

Host generators (numpy) build the small CPU-checkable cases; device
generators (torch, on the GPU) build the full-size inputs directly in HBM so
the timed region starts with resident data.  Every generator is
deterministic given its seed, so GPU and CPU arms see identical inputs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

KEY_RANGE = 1 << 20  # config 1 keys uniform in [-2^20, 2^20)^3

# ----------------------------------------------------------------- config 1


def config1_keys(seed: int = 0):
    """80,000 distinct int3 keys + 20,000 duplicates drawn from them, shuffled
    (100,000 ops, ~20% duplicates), and 100,000 keys guaranteed absent."""
    rng = np.random.default_rng(seed)
    raw = rng.integers(-KEY_RANGE, KEY_RANGE, (90_000, 3), dtype=np.int64)
    _, first = np.unique(raw, axis=0, return_index=True)
    uniq = raw[np.sort(first)][:80_000]
    dups = uniq[rng.integers(0, 80_000, 20_000)]
    keys = np.concatenate([uniq, dups])[rng.permutation(100_000)].astype(np.int32)
    absent = rng.integers(-KEY_RANGE, KEY_RANGE, (100_000, 3), dtype=np.int64)
    absent[:, 0] = rng.integers(KEY_RANGE, 2 * KEY_RANGE, 100_000)  # x outside the key range
    return np.ascontiguousarray(keys), np.ascontiguousarray(absent.astype(np.int32))


def config1_mc_keys() -> np.ndarray:
    """10,000 blocks on a 25 x 20 x 20 key grid."""
    i = np.arange(10_000)
    return np.stack([i % 25, (i // 25) % 20, i // 500], axis=1).astype(np.int32)


def random_field(n_blocks: int, seed: int = 1, hole: float = 0.15):
    """(a) tsdf ~ U(-1,1), weight = U > hole (tests/test_acceptance.py:407-412)."""
    rng = np.random.default_rng(seed)
    tsdf = rng.uniform(-1, 1, (n_blocks, 512)).astype(np.float32)
    weight = (rng.random((n_blocks, 512)) > hole).astype(np.float32)
    color = rng.integers(0, 256, (n_blocks, 512, 3)).astype(np.uint8)
    return tsdf, weight, color


def _local_coords() -> np.ndarray:
    f = np.arange(512)
    return np.stack([f % 8, (f // 8) % 8, f // 64], axis=1)


def smooth_field(keys: np.ndarray, voxel: float = 0.005, mu: float = 0.06, seed: int = 2):
    """(b) plane + sphere SDF, truncated at mu, sparse surface voxels."""
    rng = np.random.default_rng(seed)
    g = (keys[:, None, :].astype(np.float64) * 8 + _local_coords()[None]) + 0.5
    p = g * voxel
    ext = keys.max(axis=0).astype(np.float64) * 8 * voxel
    centre = ext / 2
    sphere = np.linalg.norm(p - centre, axis=-1) - 0.3 * ext.min()
    plane = p[..., 1] - 0.3 * ext[1]
    sdf = np.minimum(sphere, plane)
    tsdf = np.clip(sdf / mu, -1, 1).astype(np.float32)
    weight = np.where(np.abs(sdf) < mu, 1.0 + (rng.random(sdf.shape) * 127).astype(np.float32), 0.0)
    color = rng.integers(0, 256, keys.shape[:1] + (512, 3)).astype(np.uint8)
    return tsdf, weight.astype(np.float32), color


# ----------------------------------------------------------------- config 2

MASK63 = (1 << 63) - 1
_C1 = 0x5851F42D4C957F2D & MASK63  # odd multipliers (bijective mod 2^63)
_C2 = 0x14057B7EF767814F & MASK63


def _wrap63(v: int) -> int:
    return v & MASK63


def id_to_key_np(ids: np.ndarray) -> np.ndarray:
    """Injective id -> int3 map (a bijection on 63 bits, split 3 x 21 bits)."""
    v = ids.astype(np.uint64) & np.uint64(MASK63)
    with np.errstate(over="ignore"):
        v = (v * np.uint64(_C1)) & np.uint64(MASK63)
        v ^= v >> np.uint64(29)
        v = (v * np.uint64(_C2)) & np.uint64(MASK63)
        v ^= v >> np.uint64(32)
    m = np.uint64(0x1FFFFF)
    x = (v & m).astype(np.int64) - KEY_RANGE
    y = ((v >> np.uint64(21)) & m).astype(np.int64) - KEY_RANGE
    z = ((v >> np.uint64(42)) & m).astype(np.int64) - KEY_RANGE
    return np.stack([x, y, z], axis=1).astype(np.int32)


def id_to_key_torch(ids):
    """Same map on a torch int64 tensor (device-side generator)."""
    import torch

    m63 = MASK63
    v = ids & m63
    v = (v * _signed64(_C1)) & m63
    v = v ^ (v >> 29)
    v = (v * _signed64(_C2)) & m63
    v = v ^ (v >> 32)
    m = 0x1FFFFF
    x = (v & m) - KEY_RANGE
    y = ((v >> 21) & m) - KEY_RANGE
    z = ((v >> 42) & m) - KEY_RANGE
    return torch.stack([x, y, z], dim=1).to(torch.int32)


def _signed64(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


@dataclass
class MixSpec:
    """Config 2: live keys L at load factor lf, batches of B ops,
    50% insert (40% fresh / 60% present), 30% find (50% hit), 20% erase."""

    live: int = 10_000_000
    load_factor: float = 0.7
    batch: int = 1 << 22
    bucket_frac: float = 0.5  # share of the slots in the bucket region (the reference's defaults: equal halves)

    @property
    def slots(self) -> int:
        return math.ceil(self.live / self.load_factor)

    @property
    def bucket_count(self) -> int:
        if self.bucket_frac == 0.5:
            return (self.slots + 1) // 2
        return max(1, int(round(self.slots * self.bucket_frac)))

    @property
    def excess(self) -> int:
        return self.slots - self.bucket_count

    @property
    def counts(self) -> dict[str, int]:
        B = self.batch
        ins = B // 2
        fresh = round(0.4 * ins)
        erase = fresh  # keeps the live count (and load factor) stationary
        find = B - ins - erase
        hit = find // 2
        return {"fresh": fresh, "present": ins - fresh, "hit": hit, "miss": find - hit, "erase": erase}


MISS_BASE = 1 << 61  # ids at or above this are never inserted


def mix_batch_ids(spec: MixSpec, step: int, lo: int, hi: int, gen, device):
    """One A18-compliant mixed batch on the device.

    Live ids are [lo, hi).  Erase the oldest E ids [lo, lo+E); insert fresh
    ids [hi, hi+F); present inserts and hit finds draw from [lo+E, hi)
    (live and not erased); miss finds draw from never-inserted ids.
    Returns (ids int64[B], ops uint8[B], expect uint8[B]) in shuffled order.
    """
    import torch

    c = spec.counts
    F, P, H, M, E = c["fresh"], c["present"], c["hit"], c["miss"], c["erase"]
    keep_lo = lo + E
    fresh = torch.arange(hi, hi + F, device=device, dtype=torch.int64)
    present = torch.randint(keep_lo, hi, (P,), generator=gen, device=device, dtype=torch.int64)
    hit = torch.randint(keep_lo, hi, (H,), generator=gen, device=device, dtype=torch.int64)
    miss = MISS_BASE + step * spec.batch + torch.arange(M, device=device, dtype=torch.int64)
    erase = torch.arange(lo, lo + E, device=device, dtype=torch.int64)
    ids = torch.cat([fresh, present, hit, miss, erase])
    ops = torch.cat([torch.zeros(F + P, dtype=torch.uint8, device=device),
                     torch.ones(H + M, dtype=torch.uint8, device=device),
                     torch.full((E,), 2, dtype=torch.uint8, device=device)])
    expect = torch.cat([torch.ones(F, dtype=torch.uint8, device=device),
                        torch.zeros(P, dtype=torch.uint8, device=device),
                        torch.ones(H, dtype=torch.uint8, device=device),
                        torch.zeros(M, dtype=torch.uint8, device=device),
                        torch.ones(E, dtype=torch.uint8, device=device)])
    perm = torch.randperm(spec.batch, generator=gen, device=device)
    return ids[perm], ops[perm], expect[perm]


def mix_batch_ids_np(spec: MixSpec, step: int, lo: int, hi: int, rng: np.random.Generator):
    """numpy twin of mix_batch_ids for CPU-side tests (same structure)."""
    c = spec.counts
    F, P, H, M, E = c["fresh"], c["present"], c["hit"], c["miss"], c["erase"]
    keep_lo = lo + E
    ids = np.concatenate([np.arange(hi, hi + F), rng.integers(keep_lo, hi, P), rng.integers(keep_lo, hi, H),
                          MISS_BASE + step * spec.batch + np.arange(M), np.arange(lo, lo + E)]).astype(np.int64)
    ops = np.concatenate([np.zeros(F + P), np.ones(H + M), np.full(E, 2)]).astype(np.uint8)
    expect = np.concatenate([np.ones(F), np.zeros(P), np.ones(H), np.zeros(M), np.ones(E)]).astype(np.uint8)
    perm = rng.permutation(spec.batch)
    return ids[perm], ops[perm], expect[perm]


# ----------------------------------------------------------------- config 3

@dataclass
class RoomSpec:
    """Analytic box-room interior, 16 m x 3 m x 16 m (half-extents 8, 1.5, 8),
    5 mm voxels, truncation mu = 0.06 m."""

    half: tuple = (8.0, 1.5, 8.0)
    voxel: float = 0.005
    mu: float = 0.06
    hole_fraction: float = 0.10

    @property
    def block(self) -> float:
        return 8 * self.voxel


def room_block_keys(spec: RoomSpec = RoomSpec()) -> np.ndarray:
    """Blocks whose centre lies within mu + half a block diagonal of the walls,
    in (z, y, x)-major order (x fastest): 2,080,160 for the default room."""
    b = spec.block
    thr = spec.mu + b * math.sqrt(3) / 2
    ranges = []
    for h in spec.half:
        n = int(math.ceil(h / b)) + 2
        ranges.append(np.arange(-n, n))
    kx, ky, kz = ranges
    cx = (kx + 0.5) * b
    cy = (ky + 0.5) * b
    dx = spec.half[0] - np.abs(cx)
    dy = spec.half[1] - np.abs(cy)
    out = []
    for z in kz:
        dz = spec.half[2] - abs((z + 0.5) * b)
        d = np.minimum(np.minimum(dx[None, :], dy[:, None]), dz)  # [y, x]
        yy, xx = np.nonzero(np.abs(d) <= thr)
        if len(xx):
            out.append(np.stack([kx[xx], ky[yy], np.full(len(xx), z)], axis=1))
    return np.concatenate(out).astype(np.int32)


def _mix32_torch(v):
    """32-bit integer finaliser on int64 tensors holding uint32 values."""
    v = v & 0xFFFFFFFF
    v = ((v ^ (v >> 16)) * 0x45D9F3B) & 0xFFFFFFFF
    v = ((v ^ (v >> 16)) * 0x45D9F3B) & 0xFFFFFFFF
    return v ^ (v >> 16)


def room_tsdf_rows(keys, spec: RoomSpec = RoomSpec()):
    """TSDF wire rows (uint8[N, 6144]) of the room for int32[N,3] keys (torch).

    tsdf = clamp(sdf/mu, -1, 1); weight = 0 on ~10% holes else 1..128;
    colour = hash of the global voxel coordinate.
    """
    import torch

    dev = keys.device
    f = torch.arange(512, device=dev)
    local = torch.stack([f % 8, (f // 8) % 8, f // 64], dim=1)  # [512,3]
    g = keys.to(torch.int64)[:, None, :] * 8 + local[None]  # global voxel [N,512,3]
    p = (g.to(torch.float64) + 0.5) * spec.voxel
    half = torch.tensor(spec.half, dtype=torch.float64, device=dev)
    d = (half - p.abs()).amin(dim=-1)  # interior box SDF (positive inside the room)
    tsdf = (d / spec.mu).clamp(-1, 1).to(torch.float32)
    h = _mix32_torch(g[..., 0] * 73856093 ^ g[..., 1] * 19349669 ^ g[..., 2] * 83492791)
    hole = (h % 1000) < int(spec.hole_fraction * 1000)
    weight = torch.where(hole, torch.zeros_like(tsdf), (1 + (h >> 10) % 128).to(torch.float32))
    rgb = (_mix32_torch(h + 0x9E3779B9) & 0xFFFFFF)
    N = keys.shape[0]
    rows = torch.empty((N, 512, 3), dtype=torch.int32, device=dev)
    rows[..., 0] = tsdf.view(torch.int32)
    rows[..., 1] = weight.view(torch.int32)
    rows[..., 2] = rgb.to(torch.int32)
    return rows.view(torch.uint8).reshape(N, 6144)


# ------------------------------------------------------- RC frames (room)

def look_at(eye, target, up=(0.0, -1.0, 0.0)):
    """Camera-to-world rotation whose +z looks from eye to target, +y image-down
    (the convention of geometry.Pose.look_at)."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(np.asarray(up, np.float64), fwd)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    return np.stack([right, down, fwd], axis=1)


def room_frames(n: int, width: int = 640, height: int = 480, spec: RoomSpec = RoomSpec(), seed: int = 0):
    """n RGB-D frames rendered analytically from inside the box room: the
    camera orbits the centre at 3 m and looks at the walls; depth = distance
    along the camera z axis to the first wall hit (float32, metres), colour a
    procedural pattern of the hit point.  Returns (depth [n,h,w] f32,
    color [n,h,w,3] u8, R [n,3,3] f64, t [n,3] f64, (fx, fy, cx, cy, w, h))."""
    rng = np.random.default_rng(seed)
    f = float(width)  # ~53 degree horizontal FOV (dataset.default_intrinsics)
    intr = (f, f, width / 2, height / 2, width, height)
    half = np.asarray(spec.half, np.float64)
    uu, vv = np.meshgrid(np.arange(width, dtype=np.float64), np.arange(height, dtype=np.float64))
    cam_rays = np.stack([(uu - intr[2]) / f, (vv - intr[3]) / f, np.ones_like(uu)], axis=-1).reshape(-1, 3)
    depth = np.zeros((n, height, width), np.float32)
    color = np.zeros((n, height, width, 3), np.uint8)
    Rs = np.zeros((n, 3, 3))
    ts = np.zeros((n, 3))
    for i in range(n):
        a = 2 * np.pi * i / max(n, 1) + rng.uniform(-0.05, 0.05)
        eye = np.array([3.0 * np.cos(a), rng.uniform(-0.5, 0.5), 3.0 * np.sin(a)])
        target = np.array([8.0 * np.cos(a + 0.6), rng.uniform(-1.0, 1.0), 8.0 * np.sin(a + 0.6)])
        R = look_at(eye, target)
        d = cam_rays @ R.T
        with np.errstate(divide="ignore", invalid="ignore"):
            tt = np.where(d > 0, (half - eye) / d, np.where(d < 0, (-half - eye) / d, np.inf))
        hit_t = tt.min(axis=1)
        p = eye + d * hit_t[:, None]
        depth[i] = hit_t.reshape(height, width).astype(np.float32)
        chk = ((np.floor(p[:, 0] * 2) + np.floor(p[:, 1] * 2) + np.floor(p[:, 2] * 2)) % 2).reshape(height, width)
        color[i, ..., 0] = (80 + 120 * chk).astype(np.uint8)
        color[i, ..., 1] = (np.abs(p[:, 1]).reshape(height, width) * 60 + 40).astype(np.uint8)
        color[i, ..., 2] = (np.abs(p[:, 0] + p[:, 2]).reshape(height, width) * 10 % 255).astype(np.uint8)
        Rs[i], ts[i] = R, eye
    return depth, color, Rs, ts, intr
