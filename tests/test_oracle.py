"""CPU tests: the oracle against the golden vectors recorded from the reference.

These pin the oracle (oracle/) before it is trusted as the GPU checker.
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

import oracle
from paper_1805_03709_b200 import workloads


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------------ hash

def test_hash_kat(golden):
    cases = json.loads((golden / "hash_kat.json").read_text())
    for c in cases:
        assert oracle.hash_keys([c["key"]], c["n"])[0] == c["bucket"], c
    # the reference test-suite KATs (tests/test_concurrent_hash.py:38-58)
    assert oracle.hash_keys([(1, 2, 3)], 1 << 20)[0] == 363058
    assert oracle.hash_keys([(1, 0, 0)], 1 << 30)[0] == 73856093
    assert oracle.hash_keys([(-1, 0, 0)], 97)[0] == ((1 << 32) - 73856093) % 97


def test_scalar_hash_key_matches_golden(golden):
    from paper_1805_03709_b200.concurrent_hash import hash_key

    for c in json.loads((golden / "hash_kat.json").read_text()):
        assert hash_key(tuple(c["key"]), c["n"]) == c["bucket"]


@pytest.mark.parametrize("name", ["rand42", "chain"])
def test_sequences_positions_bit_exact(golden, name):
    sc = json.loads((golden / "hash_seq.json").read_text())[name]
    t = oracle.OracleHashSet(sc["n"], sc["excess"])
    keys = np.asarray(sc["keys"], np.int32)
    ops = np.asarray(sc["ops"], np.uint8)
    res, pos, fail = t.apply_batch(keys, ops)
    assert fail == -1
    assert res.tolist() == sc["res"]
    assert pos.tolist() == sc["pos"]  # sequential replay: positions bit-exact too
    k, p = t.snapshot()
    assert k.tolist() == sc["final"]["keys"]
    assert p.tolist() == sc["final"]["pos"]
    occ, nxt = t.raw()
    assert nxt.tolist() == sc["final"]["next"]  # incl. the stale offsets of removed entries
    assert t.free_count() == len(sc["final"]["free"])


def test_capacity_exhaustion(golden):
    sc = json.loads((golden / "hash_seq.json").read_text())["capacity"]
    t = oracle.OracleHashSet(1, 2)
    created, index, fail = t.insert_batch([(0, 0, 0), (1, 0, 0), (2, 0, 0), (3, 0, 0)])
    assert sc["raised"] and fail == 3
    k, _ = t.snapshot()
    assert sorted(map(tuple, k.tolist())) == sorted(map(tuple, sc["final"]["keys"]))


def test_config1_digests(golden):
    g = json.loads((golden / "config1_hash.json").read_text())
    keys, absent = workloads.config1_keys()
    assert sha(keys) == g["keys_sha"] and sha(absent) == g["absent_sha"]
    t = oracle.OracleHashSet(1 << 17, 1 << 17)
    created, ipos, fail = t.insert_batch(keys)
    assert fail == -1
    assert int(created.sum()) == g["created_sum"] == 80_000
    assert sha(created) == g["created_sha"]
    assert sha(ipos) == g["insert_pos_sha"]
    found, fpos = t.find_batch(np.concatenate([keys, absent]))
    assert sha(found) == g["found_sha"] and sha(fpos) == g["find_pos_sha"]
    k, _ = t.snapshot()
    assert sha(k[np.lexsort(k.T[::-1])]) == g["snapshot_sorted_sha"]
    erased, _ = t.erase_batch(keys)
    assert sha(erased) == g["erased_sha"] and int(erased.sum()) == 80_000
    assert t.size() == g["final_size"] == 0


def test_parallel_mode_matches_sequential_on_a18_batches():
    spec = workloads.MixSpec(live=20_000, load_factor=0.7, batch=1 << 13)
    rng = np.random.default_rng(3)
    seq = oracle.OracleHashSet(spec.bucket_count, spec.excess)
    par = oracle.OracleHashSet(spec.bucket_count, spec.excess)
    init = workloads.id_to_key_np(np.arange(spec.live))
    seq.insert_batch(init)
    par.insert_batch_mt(init, 4)
    lo, hi = 0, spec.live
    for step in range(4):
        ids, ops, expect = workloads.mix_batch_ids_np(spec, step, lo, hi, rng)
        keys = workloads.id_to_key_np(ids)
        r1, _, f1 = seq.apply_batch(keys, ops)
        r2, _, f2 = par.apply_batch(keys, ops, threads=4)
        assert f1 == f2 == -1
        assert np.array_equal(r1, expect) and np.array_equal(r2, expect)
        lo += spec.counts["erase"]
        hi += spec.counts["fresh"]
    a, _ = seq.snapshot()
    b, _ = par.snapshot()
    assert sorted(map(tuple, a.tolist())) == sorted(map(tuple, b.tolist()))
    assert seq.size() == par.size() == spec.live


def test_id_to_key_injective():
    ids = np.arange(200_000, dtype=np.int64) * 7919
    k = workloads.id_to_key_np(ids)
    assert len(np.unique(k, axis=0)) == len(ids)
    assert k.min() >= -(1 << 20) and k.max() < (1 << 20)


# ------------------------------------------------------------------- MC

def test_mc_random_fields_match_reference(golden):
    d = np.load(golden / "mc_random.npz")
    pool = oracle.make_pool(d["tsdf"], d["weight"], d["color"])
    nbr = oracle.neighbor_table(d["mc_keys"], d["tsdf_keys"])
    mc, q, counts = oracle.mc_encode(pool, nbr)
    assert np.array_equal(mc, d["mc"])
    assert np.array_equal(counts, (mc.reshape(-1, 512, 4)[..., 0] != 0).sum(1))


def test_mc_numpy_restatement_matches_reference(golden):
    d = np.load(golden / "mc_random.npz")
    blocks = {tuple(k): (d["tsdf"][i], d["weight"][i], d["color"][i]) for i, k in enumerate(d["tsdf_keys"].tolist())}
    for i, k in enumerate(d["mc_keys"].tolist()[:20]):
        assert oracle.mc_encode_numpy(k, blocks.get) == d["mc"][i].tobytes()


def test_mc_edge_cases(golden):
    cases = json.loads((golden / "mc_edge.json").read_text())
    for c in cases:
        t0, w0 = float(c["tsdf0"]), float(c["weight0"])
        tsdf = np.full((8, 512), 0.5, np.float32)
        weight = np.ones((8, 512), np.float32)
        color = np.full((8, 512, 3), 7, np.uint8)
        tsdf[0, 1] = -0.5
        tsdf[0, 0] = np.float32(t0)
        weight[0, 0] = np.float32(w0)
        pool = oracle.make_pool(tsdf, weight, color)
        keys = [(c_ & 1, (c_ >> 1) & 1, (c_ >> 2) & 1) for c_ in range(8)]
        nbr = oracle.neighbor_table([(0, 0, 0)], keys)
        mc, _, _ = oracle.mc_encode(pool, nbr)
        assert mc[0, 0] == c["index0"], c
        assert hashlib.sha256(mc[0].tobytes()).hexdigest() == c["mc_sha"], c


def test_mc_sphere_reproduces_manifest_digest(golden):
    d = np.load(golden / "mc_sphere.npz")
    meta = json.loads((golden / "mc_sphere.json").read_text())
    pool = oracle.make_pool(d["tsdf"], d["weight"], d["color"])
    nbr = oracle.neighbor_table(d["keys"], d["keys"])
    mc, _, _ = oracle.mc_encode(pool, nbr, threads=4)
    assert len(d["keys"]) == meta["model_blocks"] == 760
    assert hashlib.sha256(mc.tobytes()).hexdigest() == meta["model_sha256"]
    assert meta["model_sha256"] == "a02f2627fe3e61d6fc9c45566566a5bafd53ce83da92da9f9669dc2b7ccfe052"


def test_quantise_kats():
    f = np.float32
    cases = [  # (tsdf, weight, q) -- normative A17 known answers
        (0.0, 1.0, 0), (-0.0, 1.0, 0), (1.0, 1.0, 127), (-1.0, 1.0, -127),
        (0.5 / 127, 1.0, 0), (1.5 / 127, 1.0, 2), (-0.5 / 127, 1.0, 0), (-1.5 / 127, 1.0, -2),
        (2.5 / 127, 1.0, 2), (np.nan, 1.0, -128), (np.inf, 1.0, 127), (-np.inf, 1.0, -127),
        (1e-45, 1.0, 0), (-1e-45, 1.0, 0), (0.3, 0.0, -128), (0.3, -1.0, -128), (0.3, np.nan, -128),
        (0.3, 1e-45, 38), (2.0, 5.0, 127), (-3.0, 5.0, -127),
    ]
    for t, w, q in cases:
        assert int(oracle.lib().om_quantise(f(t), f(w))) == q, (t, w)
        assert int(oracle.quantise(f(t), f(w))) == q, (t, w)
    rng = np.random.default_rng(0)
    t = rng.uniform(-1.5, 1.5, 100_000).astype(np.float32)
    w = (rng.random(100_000) > 0.2).astype(np.float32)
    got = np.array([oracle.lib().om_quantise(a, b) for a, b in zip(t[:2000], w[:2000])], np.int8)
    assert np.array_equal(got, oracle.quantise(t[:2000], w[:2000]))


def test_compaction_scatter_back(golden):
    d = np.load(golden / "mc_random.npz")
    offsets, flat, cells = oracle.mc_compact(d["mc"])
    back = np.zeros_like(d["mc"]).view(np.uint32).reshape(len(d["mc"]), 512)
    for i in range(len(d["mc"])):
        a, b = int(offsets[i]), int(offsets[i + 1])
        back[i, flat[a:b]] = cells[a:b]
        assert np.all(np.diff(flat[a:b].astype(np.int64)) > 0)
    assert np.array_equal(back.view(np.uint8).reshape(d["mc"].shape), d["mc"])


# ----------------------------------------------------------- stream sets

def test_stream_oracle_matches_reference(golden):
    g = json.loads((golden / "stream_seq.json").read_text())
    for name in ("fifo_example", "random"):
        ss = oracle.OracleStreamSet()
        for op, arg, want in g[name]:
            if op in ("insert", "remove"):
                assert getattr(ss, op)(tuple(arg)) == want
            elif op == "insert_many":
                assert ss.insert_many([tuple(a) for a in arg]) == want
            else:
                assert [list(k) for k in ss.extract_ordered(arg)] == want
    assert sorted(list(k) for k in ss.set) == g["random_final"]


def test_server_fanout_oracle(golden):
    g = json.loads((golden / "server_seq.json").read_text())
    d = np.load(golden / "server_blocks.npz")
    clients = [oracle.OracleStreamSet() for _ in range(3)]
    mc_keys: set = set()
    for step, entry in enumerate(g["steps"]):
        upd = d["keys"][d["step"] == step].tolist()
        assert upd == entry["updated"]
        affected = oracle.affected_dedup(upd)
        mc_keys.update(affected)
        for c, ss in enumerate(clients):
            before = len(ss.order)
            ss.insert_many(affected)
            assert [list(k) for k in list(ss.order)[before:]] == entry["appended"][c]
            assert sorted(list(k) for k in ss.set) == entry["pending"][c]
        if "pending_after_extract_c1" in entry:
            # extract_random picks a nondeterministic subset: adopt the reference's
            keep = {tuple(k) for k in entry["pending_after_extract_c1"]}
            clients[1].set &= keep
        if "reset" in entry:
            for v in entry["reset"]:
                mc_keys.discard(tuple(v))
                for ss in clients:
                    ss.remove(tuple(v))
            for c, ss in enumerate(clients):
                assert sorted(list(k) for k in ss.set) == entry["pending_after_reset"][c]
    assert sorted(list(k) for k in mc_keys) == g["mc_keys"]
    assert g["fresh_pending"] == g["mc_keys"]


def test_fusion_oracle_matches_reference_sequence(golden):
    """The numpy RC-fusion restatement reproduces the recorded reference run
    (per-frame created / touched keys, final blocks) bit for bit."""
    from oracle.fusion_oracle import OracleVoxelModel

    d = np.load(golden / "fusion_sphere.npz")
    fx, fy, cx, cy, w, h = (float(v) for v in d["intr"])
    voxel, mu, maxw, stride = d["cfg"].tolist()
    m = OracleVoxelModel(voxel, mu, maxw, int(stride))
    c_off = np.concatenate([[0], np.cumsum(d["created_counts"])])
    t_off = np.concatenate([[0], np.cumsum(d["touched_counts"])])
    for f in range(8):
        R, t = d["pose"][f][:9].reshape(3, 3), d["pose"][f][9:]
        new = m.allocate(d["depth"][f], R, t, fx, fy, cx, cy)
        assert new == [tuple(k) for k in d["created"][c_off[f]:c_off[f + 1]].tolist()]
        got = m.integrate(d["depth"][f], d["color"][f], R, t, fx, fy, cx, cy)
        assert set(got) == {tuple(k) for k in d["touched"][t_off[f]:t_off[f + 1]].tolist()}
    s = np.load(golden / "mc_sphere.npz")
    keys = [tuple(k) for k in s["keys"].tolist()]
    assert sorted(m.blocks) == keys
    for i, k in enumerate(keys):
        tsdf, wt, col = m.blocks[k]
        assert np.array_equal(tsdf, s["tsdf"][i]) and np.array_equal(wt, s["weight"][i])
        assert np.array_equal(col, s["color"][i])


def test_extract_matches_reference(golden):
    """oh_extract == BlockHashSet.extract_batch (concurrent_hash.py:366-402)
    given the rotation start the reference drew (extract.json)."""
    for case in json.loads((golden / "extract.json").read_text()):
        o = oracle.OracleHashSet(64, 64)
        keys = np.array(case["inserted"], np.int32)
        o.insert_batch(keys)
        o.erase_batch(keys[:: case["removed_every"]])
        got = o.extract(case["max_n"], case["start"])
        assert got.tolist() == case["extracted"]
        snap = o.snapshot()[0]
        assert sorted(snap.tolist()) == case["remaining"]
