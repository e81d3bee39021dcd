"""numpy restatement of the reference RC fusion -- TEST INFRASTRUCTURE ONLY.

Follows VoxelModel.allocate_blocks / integrate_frame
(/root/reference/pkg/src/voxelstream/voxel_model.py:105-141, 165-299) and the
geometry helpers they use (geometry.py:93-101 pixel rays, :121-162 frustum),
with the same numpy dtypes and operation order, so on this numpy/OpenBLAS it
reproduces the reference bit for bit (pinned against
tests/golden/fusion_sphere.npz).  Blocks are kept in a dict of SoA arrays.
Used by tests/ and by bench.py's CPU baseline of the RC section.
"""

from __future__ import annotations

import numpy as np

BLOCK_EDGE = 8
EPS_FACE = 1e-6
_f = np.arange(512)
LOCAL = np.stack([_f % 8, (_f // 8) % 8, _f // 64], axis=1).astype(np.int64)


def block_keys_of_points(points: np.ndarray, block: float) -> np.ndarray:
    """Blocks containing the points plus, within EPS_FACE of a face, the
    neighbours across that face/edge/corner; unique, sorted by (x, y, z)."""
    g = points / block
    base = np.floor(g).astype(np.int64)
    frac = g - base
    tol = EPS_FACE / block
    near_lo, near_hi = frac < tol, frac > 1.0 - tol
    out = [base]
    edge = (near_lo | near_hi).any(axis=1)
    if edge.any():
        be, le, he = base[edge], near_lo[edge], near_hi[edge]
        for off in np.array(np.meshgrid([-1, 0, 1], [-1, 0, 1], [-1, 0, 1], indexing="ij")).reshape(3, -1).T:
            if not off.any():
                continue
            sel = np.ones(len(be), dtype=bool)
            for a in range(3):
                if off[a] < 0:
                    sel &= le[:, a]
                elif off[a] > 0:
                    sel &= he[:, a]
            if sel.any():
                out.append(be[sel] + off)
    keys = np.concatenate(out)
    return np.unique(keys, axis=0)


def frustum_planes(R, t, fx, fy, cx, cy, w, h, near, far) -> np.ndarray:
    corners = np.array([[(0 - cx) / fx, (0 - cy) / fy, 1.0], [(w - cx) / fx, (0 - cy) / fy, 1.0],
                        [(w - cx) / fx, (h - cy) / fy, 1.0], [(0 - cx) / fx, (h - cy) / fy, 1.0]])
    rays = corners @ R.T
    fwd = R[:, 2]
    rows = []
    for normal, point in [(fwd, t + near * fwd), (-fwd, t + far * fwd)] + \
            [(np.cross(rays[a], rays[b]), t) for a, b in ((0, 1), (1, 2), (2, 3), (3, 0))]:
        nn = normal / np.linalg.norm(normal)
        rows.append([*nn, -float(nn @ point)])
    return np.asarray(rows, dtype=np.float64)


class OracleVoxelModel:
    def __init__(self, voxel: float, mu: float, max_weight: float = 128.0, stride: int = 1) -> None:
        self.voxel, self.mu, self.max_weight, self.stride = voxel, mu, max_weight, stride
        self.block = BLOCK_EDGE * voxel
        self.blocks: dict = {}  # key -> [tsdf f32[512], weight f32[512], color u8[512,3]]

    def allocate(self, depth, R, t, fx, fy, cx, cy) -> list:
        s = self.stride
        dsub = depth[::s, ::s]
        valid = dsub > 0
        if not valid.any():
            return []
        h, w = depth.shape
        uu, vv = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
        rays = np.stack([(uu - cx) / fx, (vv - cy) / fy, np.ones_like(uu)], axis=-1)[::s, ::s][valid]
        d = dsub[valid].astype(np.float64)
        z0 = np.maximum(d - self.mu, self.voxel)
        z1 = d + self.mu
        n = int(np.ceil(2 * self.mu / self.voxel)) + 1
        ts = np.linspace(0.0, 1.0, n)
        zs = z0[:, None] + (z1 - z0)[:, None] * ts[None, :]
        pts = (rays[:, None, :] * zs[:, :, None]).reshape(-1, 3)
        world = pts @ R.T + t
        new = []
        for k in map(tuple, block_keys_of_points(world, self.block).tolist()):
            if k not in self.blocks:
                self.blocks[k] = [np.zeros(512, np.float32), np.zeros(512, np.float32), np.zeros((512, 3), np.uint8)]
                new.append(k)
        return new

    def integrate(self, depth, color, R, t, fx, fy, cx, cy) -> list:
        if not self.blocks:
            return []
        h, w = depth.shape
        keys = list(self.blocks)
        karr = np.asarray(keys, dtype=np.int64)
        planes = frustum_planes(R, t, fx, fy, cx, cy, w, h, 0.05, 20.0)
        lo = karr.astype(np.float64) * self.block
        hi = lo + self.block
        vis = np.ones(len(karr), dtype=bool)
        for pl in planes:
            v = np.where(pl[:3] >= 0, hi, lo)
            vis &= v @ pl[:3] + pl[3] >= -self.block
        sel = np.flatnonzero(vis)
        if sel.size == 0:
            return []
        karr = karr[sel]
        cen = (karr + 0.5) * self.block
        cc = (cen - t) @ R
        cz = cc[:, 2]
        with np.errstate(divide="ignore", invalid="ignore"):
            cu = np.rint(fx * cc[:, 0] / cz + cx)
            cv = np.rint(fy * cc[:, 1] / cz + cy)
        inside = (cz > 0) & (cu >= 0) & (cu < w) & (cv >= 0) & (cv < h)
        cd = np.zeros(len(karr), dtype=np.float32)
        cd[inside] = depth[cv[inside].astype(np.int64), cu[inside].astype(np.int64)]
        far = inside & (cd > 0) & (np.abs(cd - cz) > self.mu + self.block * np.sqrt(3.0))
        sel = sel[~far]
        karr = karr[~far]
        if sel.size == 0:
            return []
        coords = ((karr[:, None, :] * BLOCK_EDGE + LOCAL[None] + 0.5) * self.voxel).astype(np.float32)
        cam = ((coords.reshape(-1, 3) - t.astype(np.float32)) @ R.astype(np.float32)).reshape(len(sel), 512, 3)
        z = cam[:, :, 2]
        with np.errstate(divide="ignore", invalid="ignore"):
            u = np.rint(fx * cam[:, :, 0] / z + cx).astype(np.int32)
            v = np.rint(fy * cam[:, :, 1] / z + cy).astype(np.int32)
        ok = (z > 0) & (u >= 0) & (u < w) & (v >= 0) & (v < h)
        ui, vi = np.clip(u, 0, w - 1), np.clip(v, 0, h - 1)
        dd = depth[vi, ui]
        sdf = dd - z
        ok &= (dd > 0) & (sdf >= -self.mu)
        obs = np.clip(sdf / self.mu, -1.0, 1.0)
        smp = color[vi, ui].astype(np.float32)
        out = []
        for j, bi in enumerate(sel):
            m = ok[j]
            if not m.any():
                continue
            tsdf, wt, col = self.blocks[keys[bi]]
            w0 = wt[m]
            w1 = w0 + 1.0
            tsdf[m] = (tsdf[m] * w0 + obs[j][m].astype(np.float32)) / w1
            col[m] = np.rint((col[m].astype(np.float32) * w0[:, None] + smp[j][m]) / w1[:, None]).astype(np.uint8)
            wt[m] = np.minimum(w1, self.max_weight)
            out.append(keys[bi])
        return out
