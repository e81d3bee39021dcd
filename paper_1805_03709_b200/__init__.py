"""B200-native SLAMCast hot path: drop-in GPU replacement of the reference
``voxelstream`` block hash set/map, MC block encoder and per-client stream
sets.  Every computation runs in libvsb200.so (hand-written sm_100a CUDA,
C ABI in include/vsb200.h); there is no CPU fallback.

Public names mirror voxelstream/__init__.py:11-34 for the hot path.
"""

from ._lib import CapacityExhausted, NativeUnavailable
from .concurrent_hash import (
    BlockHashMap,
    BlockHashSet,
    BlockKey,
    FreeListStack,
    hash_key,
    hash_keys,
)
from .mc_encoding import (
    McBlock,
    McVoxel,
    affected_mc_blocks,
    apply_cutoff,
    compact,
    compute_mc_index,
    encode_blocks,
    encode_keys,
    face_packs,
    neighbors,
    pack_mc_batch,
    recompute_mc_block,
    recompute_mc_blocks,
)
from .server import GpuServerCore, StreamSet, extract_random_many, fan_out, remove_everywhere, stream_tick
from .voxel_model import BLOCK_EDGE, TsdfBlock

__all__ = [
    "BLOCK_EDGE", "BlockHashMap", "BlockHashSet", "BlockKey", "CapacityExhausted", "FreeListStack",
    "GpuServerCore", "McBlock", "McVoxel", "NativeUnavailable", "StreamSet", "TsdfBlock",
    "affected_mc_blocks", "apply_cutoff", "compact", "compute_mc_index", "encode_blocks", "encode_keys", "face_packs",
    "extract_random_many", "stream_tick", "fan_out", "hash_key", "hash_keys", "neighbors", "pack_mc_batch", "recompute_mc_block", "recompute_mc_blocks",
    "remove_everywhere",
]

__version__ = "0.1.0"
