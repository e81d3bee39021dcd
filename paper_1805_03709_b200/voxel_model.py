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
