"""GPU parity tests of the MC block encoder (+ quantised TSDF, compaction).

Bar: bit-exact MC bytes against the reference's recorded outputs and the
C oracle; quantised TSDF bit-exact against the normative oracle (A17);
compaction scatters back to the dense bytes (A19).
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

import oracle
from paper_1805_03709_b200 import workloads

pytestmark = pytest.mark.gpu


def _t(a, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def gpu_encode(pool, nbr, dev):
    """Encode through both halo paths -- scattered voxel reads and the face
    bit-packs -- which must agree byte for byte; returns the first."""
    import torch

    from paper_1805_03709_b200 import encode_blocks, face_packs

    p, nb = _t(pool, dev), _t(nbr, dev)
    mc, q, c = encode_blocks(p, nb)
    mc2, q2, c2 = encode_blocks(p, nb, faces=face_packs(p))
    assert torch.equal(mc, mc2) and torch.equal(q, q2) and torch.equal(c, c2), "face-pack halo path differs"
    return mc.cpu().numpy(), q.cpu().numpy(), c.cpu().numpy().astype(np.uint32)


def check_cells_scatter_back(mc, counts, offs, flat, cells):
    """Fused compaction (A19): every block's cells, read through its range,
    scatter back to its dense MC bytes; ranges are disjoint."""
    import torch

    n = mc.shape[0]
    counts = counts.long()
    offs = offs.long()
    total = int(counts.sum().item())
    blk = torch.repeat_interleave(torch.arange(n, device=mc.device), counts)
    start = torch.repeat_interleave(offs, counts)
    within = torch.arange(total, device=mc.device) - torch.repeat_interleave(torch.cumsum(counts, 0) - counts, counts)
    src = start + within
    assert total == 0 or int(src.max().item()) < total
    assert torch.unique(src).numel() == total  # disjoint ranges covering [0, total)
    dense = torch.zeros((n, 512), dtype=torch.int32, device=mc.device)
    f = flat[src].long() & 0xFFFF
    dense[blk, f] = cells[src]
    assert torch.equal(dense.view(torch.uint8).view(n, 2048), mc)
    # ascending flat index inside each block
    if total > 1:
        same = blk[1:] == blk[:-1]
        assert bool(torch.all(f[1:][same] > f[:-1][same]))


def table_with_pool(tsdf_keys, rows, dev, n=1 << 12, excess=1 << 12):
    """A BlockHashMap-style table whose positions index a device pool."""
    import torch

    from paper_1805_03709_b200 import BlockHashSet

    t = BlockHashSet(n, excess)
    created, pos = t.insert_keys(tsdf_keys)
    t.check_capacity()
    pool = torch.zeros((t.capacity, 6144), dtype=torch.uint8, device=dev)
    pool[pos.long()] = _t(rows, dev)
    return t, pool


def test_random_fields_vs_reference(dev, golden):
    d = np.load(golden / "mc_random.npz")
    pool = oracle.make_pool(d["tsdf"], d["weight"], d["color"])
    nbr = oracle.neighbor_table(d["mc_keys"], d["tsdf_keys"])
    mc, q, counts = gpu_encode(pool, nbr, dev)
    assert np.array_equal(mc, d["mc"])  # reference recompute_mc_block bytes
    omc, oq, oc = oracle.mc_encode(pool, nbr)
    assert np.array_equal(q, oq) and np.array_equal(counts, oc)


def test_fused_hash_lookup_path_vs_reference(dev, golden):
    from paper_1805_03709_b200 import encode_keys, neighbors

    d = np.load(golden / "mc_random.npz")
    rows = oracle.make_pool(d["tsdf"], d["weight"], d["color"])
    t, pool = table_with_pool(d["tsdf_keys"], rows, dev)
    mc, q, c = encode_keys(t, pool, d["mc_keys"])
    assert np.array_equal(mc.cpu().numpy(), d["mc"])
    nbr = neighbors(t, d["mc_keys"]).cpu().numpy()
    ref_nbr = oracle.neighbor_table(d["mc_keys"], d["tsdf_keys"])
    assert np.array_equal(nbr >= 0, ref_nbr >= 0)


def test_ieee_edge_cases(dev, golden):
    for c in json.loads((golden / "mc_edge.json").read_text()):
        tsdf = np.full((8, 512), 0.5, np.float32)
        weight = np.ones((8, 512), np.float32)
        color = np.full((8, 512, 3), 7, np.uint8)
        tsdf[0, 1] = -0.5
        tsdf[0, 0] = np.float32(float(c["tsdf0"]))
        weight[0, 0] = np.float32(float(c["weight0"]))
        pool = oracle.make_pool(tsdf, weight, color)
        nbr = oracle.neighbor_table([(0, 0, 0)], [(k & 1, (k >> 1) & 1, (k >> 2) & 1) for k in range(8)])
        mc, q, _ = gpu_encode(pool, nbr, dev)
        assert mc[0, 0] == c["index0"], c
        assert hashlib.sha256(mc[0].tobytes()).hexdigest() == c["mc_sha"], c
        assert np.array_equal(q, oracle.mc_encode(pool, nbr)[1])


def test_fused_sphere_reproduces_manifest_model_sha256(dev, golden):
    """The reference's pipeline golden (pkg/fixtures/protocol/manifest.json):
    760 sorted-key MC payloads of the fused sphere hash to model_sha256."""
    from paper_1805_03709_b200 import encode_keys

    d = np.load(golden / "mc_sphere.npz")
    meta = json.loads((golden / "mc_sphere.json").read_text())
    rows = oracle.make_pool(d["tsdf"], d["weight"], d["color"])
    t, pool = table_with_pool(d["keys"], rows, dev)
    mc, _, _ = encode_keys(t, pool, d["keys"])
    assert hashlib.sha256(mc.cpu().numpy().tobytes()).hexdigest() == meta["model_sha256"]
    from paper_1805_03709_b200 import face_packs

    mc2, _, _ = encode_keys(t, pool, d["keys"], faces=face_packs(pool))
    assert hashlib.sha256(mc2.cpu().numpy().tobytes()).hexdigest() == meta["model_sha256"]
    # fused compaction + output rows (the server path): same bytes at the rows
    import torch

    rows = torch.arange(len(d["keys"]) - 1, -1, -1, dtype=torch.int32, device=dev)
    mpool = torch.zeros((len(d["keys"]), 2048), dtype=torch.uint8, device=dev)
    qpool = torch.zeros((len(d["keys"]), 512), dtype=torch.int8, device=dev)
    _, _, c3, (offs, flat, cells, cur) = encode_keys(t, pool, d["keys"], mc=mpool, q=qpool, out_rows=rows,
                                                     cells=True, faces=face_packs(pool))
    mc3 = mpool.flip(0)
    assert hashlib.sha256(mc3.cpu().numpy().tobytes()).hexdigest() == meta["model_sha256"]
    check_cells_scatter_back(mc3, c3, offs, flat, cells)


@pytest.mark.parametrize("field", ["random", "smooth"])
def test_config1_mc_10k_blocks_vs_oracle(dev, field):
    keys = workloads.config1_mc_keys()
    if field == "random":
        tsdf, weight, color = workloads.random_field(len(keys))
    else:
        tsdf, weight, color = workloads.smooth_field(keys)
    pool = oracle.make_pool(tsdf, weight, color)
    # MC keys = the TSDF keys plus the -1 shell (absent centres -> zero blocks)
    mkeys = np.concatenate([keys, keys[:200] - 1])
    nbr = oracle.neighbor_table(mkeys, keys)
    mc, q, counts = gpu_encode(pool, nbr, dev)
    omc, oq, oc = oracle.mc_encode(pool, nbr, threads=8)
    assert np.array_equal(mc, omc)
    assert np.array_equal(q, oq)
    assert np.array_equal(counts, oc)
    assert counts.sum() > 0


def test_compaction_vs_oracle_and_scatter_back(dev):
    import torch

    from paper_1805_03709_b200 import compact, encode_blocks

    keys = workloads.config1_mc_keys()[:3000]
    tsdf, weight, color = workloads.random_field(len(keys), seed=5)
    pool = oracle.make_pool(tsdf, weight, color)
    nbr = oracle.neighbor_table(keys, keys)
    mc, _, counts = encode_blocks(_t(pool, dev), _t(nbr, dev))
    offsets, flat, cells = compact(mc, counts)
    oo, of, oc = oracle.mc_compact(mc.cpu().numpy())
    assert np.array_equal(offsets.cpu().numpy().astype(np.uint64), oo)
    assert np.array_equal(flat.cpu().numpy().view(np.uint16), of)
    assert np.array_equal(cells.cpu().numpy().view(np.uint32), oc)
    dense = torch.zeros((len(keys), 512), dtype=torch.int32, device=dev)
    blk = torch.repeat_interleave(torch.arange(len(keys), device=dev), counts.long())
    dense[blk, flat.long() & 0xFFFF] = cells
    assert torch.equal(dense.view(torch.uint8).reshape(mc.shape), mc)


def test_recompute_mc_block_api_with_host_blocks(dev, golden):
    from paper_1805_03709_b200 import TsdfBlock, recompute_mc_block, recompute_mc_blocks

    d = np.load(golden / "mc_random.npz")
    blocks = {}
    for i, k in enumerate(d["tsdf_keys"].tolist()):
        b = TsdfBlock(tuple(k))
        b.tsdf, b.weight, b.color = d["tsdf"][i], d["weight"][i], d["color"][i]
        blocks[tuple(k)] = b
    keys = [tuple(k) for k in d["mc_keys"].tolist()]
    out = recompute_mc_blocks(keys, blocks.get)
    assert b"".join(m.to_bytes() for m in out) == d["mc"].tobytes()
    one = recompute_mc_block(keys[5], blocks.get)
    assert one.to_bytes() == d["mc"][5].tobytes()
    assert recompute_mc_block((40, 40, 40), blocks.get).is_empty()


def test_room_sample_vs_oracle(dev):
    """Config 3 geometry: the room corner around x = z = -8 m (walls, floor,
    ceiling and their edges, ~50k blocks), GPU vs oracle."""
    import torch

    from paper_1805_03709_b200 import encode_keys

    keys = workloads.room_block_keys()
    keys = keys[(keys[:, 0] <= -160) & (keys[:, 2] <= -160)]
    kt = torch.from_numpy(keys).to(dev)
    rows = workloads.room_tsdf_rows(kt)
    t, pool = table_with_pool(keys, rows.cpu().numpy(), dev, n=1 << 16, excess=1 << 16)
    mc, q, c = encode_keys(t, pool, keys)
    from paper_1805_03709_b200 import face_packs

    # face packs maintained for the written rows only (the rest stay zero and
    # are never looked up): same bytes
    _, pos = t.find_keys(keys)
    mc2, q2, c2 = encode_keys(t, pool, keys, faces=face_packs(pool, rows=pos))
    assert torch.equal(mc, mc2) and torch.equal(q, q2) and torch.equal(c, c2)
    for fc in (None, face_packs(pool, rows=pos)):  # fused compaction, both halo paths
        mc3, q3, c3, (offs, flat, cells, cur) = encode_keys(t, pool, keys, faces=fc, cells=True)
        assert torch.equal(mc, mc3) and torch.equal(q, q3) and torch.equal(c, c3)
        assert int(cur.item()) == int(c.sum().item())
        check_cells_scatter_back(mc, c3, offs, flat, cells)
    rows_np = rows.cpu().numpy()
    nbr = oracle.neighbor_table(keys, keys)
    omc, oq, oc = oracle.mc_encode(rows_np, nbr, threads=8)
    assert np.array_equal(mc.cpu().numpy(), omc)
    assert np.array_equal(q.cpu().numpy(), oq)
    assert np.array_equal(c.cpu().numpy().astype(np.uint32), oc)
    assert oc.sum() > 0


def test_face_packs_track_row_updates(dev):
    """Packs recomputed for changed rows only keep the face-pack encode equal
    to the scattered-halo encode (the ingest contract of vs_mc_faces)."""
    import torch

    from paper_1805_03709_b200 import encode_blocks, face_packs

    keys = workloads.config1_mc_keys()[:2000]
    tsdf, weight, color = workloads.random_field(len(keys), seed=9)
    pool = _t(oracle.make_pool(tsdf, weight, color), dev)
    nbr = _t(oracle.neighbor_table(keys, keys), dev)
    faces = face_packs(pool)
    rng = np.random.default_rng(4)
    for step in range(3):
        rows = torch.from_numpy(rng.choice(len(keys), 300, replace=False).astype(np.int32)).to(dev)
        t2, w2, c2 = workloads.random_field(300, seed=100 + step)
        pool[rows.long()] = _t(oracle.make_pool(t2, w2, c2), dev)
        face_packs(pool, rows=rows, faces=faces)
        a = encode_blocks(pool, nbr)
        b = encode_blocks(pool, nbr, faces=faces)
        assert all(torch.equal(x, y) for x, y in zip(a, b)), step


@pytest.mark.gpu
def test_ticketed_work_distribution_vs_oracle(dev):
    """Launches of >= 4 lookup batches per CTA take their blocks from the
    per-stream ticket counter (mc.cu launch_mc_t); 114k room blocks exercise
    that path for every encoder variant, twice on one stream (the last CTA
    re-zeroes the counter) and once on a second stream, against the oracle."""
    import torch

    from paper_1805_03709_b200 import encode_blocks, encode_keys, face_packs

    keys = workloads.room_block_keys()
    keys = keys[(keys[:, 0] <= -120) & (keys[:, 2] <= -120)]
    assert len(keys) > 148 * 10 * 16 * 4  # above the ticket threshold of a full grid
    kt = torch.from_numpy(keys).to(dev)
    rows = workloads.room_tsdf_rows(kt)
    t, pool = table_with_pool(keys, rows.cpu().numpy(), dev, n=1 << 17, excess=1 << 17)
    nbr = oracle.neighbor_table(keys, keys)
    omc, oq, oc = oracle.mc_encode(rows.cpu().numpy(), nbr, threads=8)
    _, pos = t.find_keys(keys)
    fp = face_packs(pool, rows=pos)
    side = torch.cuda.Stream(dev)
    nbr_rows = torch.from_numpy(np.where(nbr >= 0, pos.cpu().numpy()[np.maximum(nbr, 0)], -1).astype(np.int32)).to(dev)
    for run in range(3):
        with torch.cuda.stream(side if run == 2 else torch.cuda.current_stream(dev)):
            outs = [encode_keys(t, pool, keys), encode_keys(t, pool, keys, faces=fp), encode_blocks(pool, nbr_rows)]
            mc4, q4, c4, (offs, flat, cells, cur) = encode_keys(t, pool, keys, cells=True)
        if run == 2:  # a second stream's launches, queued while the side stream's may still run
            outs.append(encode_blocks(pool, nbr_rows))
        torch.cuda.synchronize()
        for mc, q, c in outs + [(mc4, q4, c4)]:
            assert np.array_equal(mc.cpu().numpy(), omc)
            assert np.array_equal(q.cpu().numpy(), oq)
            assert np.array_equal(c.cpu().numpy().astype(np.uint32), oc)
        assert int(cur.item()) == int(oc.sum())
        check_cells_scatter_back(mc4, c4, offs, flat, cells)
