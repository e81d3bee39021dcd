"""Edge cases on the GPU path: empty and ragged inputs, limits, invalid
arguments (ValueError like concurrent_hash.py:96-101), absent neighbours."""

from __future__ import annotations

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_empty_batches_everywhere(dev):
    import torch

    from paper_1805_03709_b200 import (BlockHashSet, StreamSet, compact, encode_blocks, encode_keys,
                                       extract_random_many, fan_out, hash_keys, pack_mc_batch, remove_everywhere)

    s = BlockHashSet(16, 16)
    empty = torch.empty((0, 3), dtype=torch.int32, device=dev)
    c, i = s.insert_keys(empty)
    assert c.numel() == 0 and i.numel() == 0
    assert s.find_keys(empty)[0].numel() == 0
    assert s.erase_keys(empty)[0].numel() == 0
    assert s.apply(empty, torch.empty(0, dtype=torch.uint8, device=dev))[0].numel() == 0
    assert s.extract_batch(0) == [] and s.extract_batch(5) == []
    assert s.snapshot_keys() == [] and s.approx_size() == 0
    assert hash_keys(empty, 97).numel() == 0
    pool = torch.zeros((4, 6144), dtype=torch.uint8, device=dev)
    mc, q, cnt = encode_blocks(pool, torch.empty((0, 8), dtype=torch.int32, device=dev))
    assert mc.shape == (0, 2048) and q.shape == (0, 512)
    mc, q, cnt = encode_keys(s, pool, empty)
    assert mc.shape[0] == 0
    off, flat, cells = compact(mc, cnt)
    assert off.tolist() == [0] and flat.numel() == 0
    payload = pack_mc_batch(empty, torch.empty(0, dtype=torch.int32, device=dev), torch.zeros((1, 2048), dtype=torch.uint8, device=dev))
    assert payload.cpu().tolist() == [0, 0, 0, 0]
    sets = [StreamSet(16, 16) for _ in range(2)]
    assert fan_out(sets, empty) == [0, 0]
    remove_everywhere(sets, empty)
    k, n = extract_random_many(sets, 8)
    assert n.tolist() == [0, 0]
    assert sets[0].extract_ordered(5) == []


def test_invalid_sizes_raise_valueerror(dev):
    from paper_1805_03709_b200 import BlockHashSet

    for args in [(0, 4), (4, 0), (-1, 4), (4, 1 << 29), ((1 << 31) - 8, 8)]:
        with pytest.raises(ValueError):
            BlockHashSet(*args)
    with pytest.raises(ValueError):
        BlockHashSet(64, 64, lock_stripes=6)


def test_extreme_keys_and_tiny_tables(dev):
    """Full int32 key range (no sentinel), 1-bucket tables (one long chain)."""
    from paper_1805_03709_b200 import BlockHashSet

    lo, hi = -(2 ** 31), 2 ** 31 - 1
    keys = [(lo, lo, lo), (hi, hi, hi), (lo, hi, 0), (0, 0, 0), (-1, -1, -1), (hi, lo, hi)]
    s = BlockHashSet(1, 8)
    created, idx = s.insert_keys(keys)
    assert created.sum().item() == 6 and len(set(idx.tolist())) == 6
    assert all(k in s for k in keys)
    assert (5, 5, 5) not in s
    erased, _ = s.erase_keys(keys[::2])
    assert erased.tolist() == [1, 1, 1]
    assert sorted(s.snapshot_keys()) == sorted(keys[1::2])
    a = s.audit()
    assert a["duplicates"] == 0 and a["free"] + a["reachable_excess"] == 8


def test_mc_isolated_blocks_and_absent_neighbours(dev):
    """Blocks without any neighbour: every +face cube is unobserved -> 0
    (measured reference behaviour); absent centres -> zeros."""
    import torch

    from paper_1805_03709_b200 import encode_blocks

    tsdf, weight, color = __import__("paper_1805_03709_b200.workloads", fromlist=["x"]).random_field(6, seed=4, hole=0.0)
    rows = oracle.make_pool(tsdf, weight, color)
    nbr = np.full((8, 8), -1, np.int32)
    nbr[:6, 0] = np.arange(6)
    mc, q, cnt = encode_blocks(torch.from_numpy(rows).cuda(), torch.from_numpy(nbr).cuda())
    omc, oq, oc = oracle.mc_encode(rows, nbr)
    assert np.array_equal(mc.cpu().numpy(), omc) and np.array_equal(q.cpu().numpy(), oq)
    grid = mc.cpu().numpy().reshape(8, 8, 8, 8, 4)[..., 0]  # [blk, z, y, x]
    assert not grid[:, 7].any() and not grid[:, :, 7].any() and not grid[:, :, :, 7].any()
    assert not mc[6:].any() and (q[6:] == -128).all()


def test_misaligned_pool_is_rejected(dev):
    import torch

    from paper_1805_03709_b200 import _lib

    buf = torch.zeros(6144 * 2 + 16, dtype=torch.uint8, device=dev)
    nbr = torch.full((1, 8), -1, dtype=torch.int32, device=dev)
    st = _lib.load().vs_mc_encode(_lib.ctypes.c_void_p(buf.data_ptr() + 4), None, _lib.ptr(nbr), 1, None, None,
                                  None, _lib.stream_of(dev))
    assert st == _lib.VS_ERR_INVALID
    # misaligned face packs likewise
    st = _lib.load().vs_mc_encode(_lib.ptr(buf), _lib.ctypes.c_void_p(buf.data_ptr() + 4), _lib.ptr(nbr), 1, None,
                                  None, None, _lib.stream_of(dev))
    assert st == _lib.VS_ERR_INVALID
