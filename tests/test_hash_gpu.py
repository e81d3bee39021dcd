"""GPU parity tests of the block hash set/map against the oracle and the
golden vectors recorded from the reference (tests/golden/).

Parity rules:
  * per-op result flags (created / found / erased) are bit-exact against a
    sequential replay for batches that follow the A18 rule;
  * entry positions are compared canonically: every op on one key returns
    the same position, distinct live keys have distinct positions in
    [0, capacity) -- the concrete values depend on thread interleaving;
  * the final key set, sorted, is bit-exact.
"""

from __future__ import annotations

import hashlib
import json
import threading

import numpy as np
import pytest

import oracle
from paper_1805_03709_b200 import workloads

pytestmark = pytest.mark.gpu


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sorted_keys(k: np.ndarray) -> np.ndarray:
    k = np.asarray(k).reshape(-1, 3)
    return k[np.lexsort(k.T[::-1])]


def canonical_positions_ok(keys: np.ndarray, pos: np.ndarray, ok: np.ndarray, capacity: int) -> None:
    """Same key -> same position; different keys -> different positions."""
    keys = np.asarray(keys).reshape(-1, 3)[ok]
    pos = np.asarray(pos)[ok]
    assert pos.min() >= 0 and pos.max() < capacity
    _, kid = np.unique(keys, axis=0, return_inverse=True)
    kid = kid.reshape(-1)
    first_pos = {}
    for k, p in zip(kid.tolist(), pos.tolist()):
        assert first_pos.setdefault(k, p) == p
    assert len(set(first_pos.values())) == len(first_pos)


def audit_clean(s, live: int) -> None:
    a = s.audit()
    assert a["duplicates"] == 0 and a["unreachable_live"] == 0 and a["free_reachable"] == 0, a
    assert a["live"] == live == s.approx_size(), a
    assert a["free"] + a["reachable_excess"] == s.excess_capacity, a  # free-list conservation


def test_hash_keys_match_golden(dev, golden):
    import torch

    from paper_1805_03709_b200 import hash_keys

    cases = json.loads((golden / "hash_kat.json").read_text())
    for n in sorted({c["n"] for c in cases}):
        sub = [c for c in cases if c["n"] == n]
        got = hash_keys(torch.tensor([c["key"] for c in sub], dtype=torch.int32), n).cpu().tolist()
        assert got == [c["bucket"] for c in sub], n


@pytest.mark.parametrize("name", ["rand42", "chain"])
def test_reference_sequence_per_op(dev, golden, name):
    """Replay the reference's recorded op sequence one op per launch."""
    from paper_1805_03709_b200 import BlockHashSet

    sc = json.loads((golden / "hash_seq.json").read_text())[name]
    s = BlockHashSet(sc["n"], sc["excess"])
    pos_of = {}
    for op, key, want in zip(sc["ops"], sc["keys"], sc["res"]):
        key = tuple(key)
        if op == 0:
            p, created = s._insert_pos(key)
            assert created == bool(want)
            assert pos_of.setdefault(key, p) == p  # stable while present
        elif op == 1:
            assert (key in s) == bool(want)
        else:
            assert s.remove(key) == bool(want)
            if want:
                pos_of.pop(key, None)
    got = sorted(s.snapshot_keys())
    assert got == sorted(tuple(k) for k in sc["final"]["keys"])
    audit_clean(s, len(got))


def test_config1_bit_exact_against_reference_digests(dev, golden):
    """BASELINE config 1 (100k keys, ~20% dups): batched GPU ops give the
    reference's per-op flags bit for bit (digests recorded from it)."""
    from paper_1805_03709_b200 import BlockHashSet

    g = json.loads((golden / "config1_hash.json").read_text())
    keys, absent = workloads.config1_keys()
    assert sha(keys) == g["keys_sha"]
    s = BlockHashSet(1 << 17, 1 << 17)
    created, index = s.insert_keys(keys)
    s.check_capacity()
    created, index = created.cpu().numpy(), index.cpu().numpy()
    assert sha(created) == g["created_sha"] and int(created.sum()) == 80_000
    canonical_positions_ok(keys, index, np.ones(len(keys), bool), s.capacity)
    probe = np.concatenate([keys, absent])
    found, fidx = s.find_keys(probe)
    found, fidx = found.cpu().numpy(), fidx.cpu().numpy()
    assert sha(found) == g["found_sha"]
    assert np.array_equal(fidx[: len(keys)], index)  # finds agree with insert positions
    snap = s.snapshot_tensor()[0].cpu().numpy()
    assert sha(sorted_keys(snap)) == g["snapshot_sorted_sha"]
    audit_clean(s, 80_000)
    erased, _ = s.erase_keys(keys)
    assert sha(erased.cpu().numpy()) == g["erased_sha"]
    assert s.approx_size() == 0
    audit_clean(s, 0)


def test_mixed_batches_match_oracle_and_expectation(dev):
    """Config-2 workload shape at reduced size: per-op results bit-exact vs
    the analytic expectation and vs the sequential oracle, LF stationary."""
    import torch

    from paper_1805_03709_b200 import BlockHashSet

    spec = workloads.MixSpec(live=200_000, load_factor=0.7, batch=1 << 16)
    s = BlockHashSet(spec.bucket_count, spec.excess)
    o = oracle.OracleHashSet(spec.bucket_count, spec.excess)
    init = workloads.id_to_key_np(np.arange(spec.live))
    s.insert_keys(init)
    s.check_capacity()
    o.insert_batch(init)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    lo, hi = 0, spec.live
    for step in range(6):
        ids, ops, expect = workloads.mix_batch_ids(spec, step, lo, hi, gen, dev)
        keys = workloads.id_to_key_torch(ids)
        res, idx = s.apply(keys, ops)
        s.check_capacity()
        res = res.cpu().numpy()
        assert np.array_equal(res, expect.cpu().numpy()), step
        ores, _, fail = o.apply_batch(keys.cpu().numpy(), ops.cpu().numpy())
        assert fail == -1 and np.array_equal(res, ores)
        ok = (res == 1) | (ops.cpu().numpy() == 0)
        canonical_positions_ok(keys.cpu().numpy(), idx.cpu().numpy(), ok & (ops.cpu().numpy() != 2), s.capacity)
        lo += spec.counts["erase"]
        hi += spec.counts["fresh"]
        assert s.approx_size() == spec.live
    a = sorted_keys(s.snapshot_tensor()[0].cpu().numpy())
    b = sorted_keys(o.snapshot()[0])
    assert np.array_equal(a, b)
    audit_clean(s, spec.live)


def test_same_key_from_many_threads_single_entry(dev):
    """tests/test_concurrent_hash.py:100-114 and test_acceptance.py:279-321,
    GPU form: thousands of threads insert the same keys in one launch."""
    import torch

    from paper_1805_03709_b200 import BlockHashSet

    s = BlockHashSet(8, 4096)
    base = np.array([[3, 1, 4]], np.int32)
    keys = np.repeat(base, 20_000, axis=0)
    created, idx = s.insert_keys(keys)
    c = created.cpu().numpy()
    assert c[0] == 1 and c.sum() == 1  # the lowest op index creates
    assert len(set(idx.cpu().tolist())) == 1
    # 1000 keys x 64 copies, shuffled, into a tiny bucket array (long chains)
    rng = np.random.default_rng(0)
    k = np.stack([np.arange(1000), np.zeros(1000), np.ones(1000)], 1).astype(np.int32)
    many = np.repeat(k, 64, axis=0)[rng.permutation(64_000)]
    created, idx = s.insert_keys(many)
    c = created.cpu().numpy()
    o = oracle.OracleHashSet(8, 4096)
    o.insert_batch(base)
    oc, _, _ = o.insert_batch(many)
    assert np.array_equal(c, oc)  # first occurrence of each key creates
    canonical_positions_ok(many, idx.cpu().numpy(), np.ones(len(many), bool), s.capacity)
    audit_clean(s, 1001)


def test_contended_insert_erase_keeps_uniqueness(dev):
    """A batch that violates A18 on purpose (inserts and erases of the same
    keys race): any linearisation is allowed, uniqueness must hold."""
    import torch

    from paper_1805_03709_b200 import BlockHashSet

    s = BlockHashSet(4, 8192)
    rng = np.random.default_rng(1)
    for _ in range(20):
        keys = np.stack([rng.integers(0, 64, 50_000), np.zeros(50_000), np.zeros(50_000)], 1).astype(np.int32)
        ops = (rng.random(50_000) < 0.3).astype(np.uint8) * 2
        s.apply(keys, torch.from_numpy(ops))
        a = s.audit()
        assert a["duplicates"] == 0 and a["unreachable_live"] == 0 and a["free_reachable"] == 0
        assert a["free"] + a["reachable_excess"] == s.excess_capacity
        assert a["live"] == s.approx_size() <= 64


def test_fresh_erase_reclaim_aba_keeps_uniqueness(dev):
    """A18-violating batches built to hit the bucket-word ABA: per bucket one
    insert of K (fresh), erases of K and several inserts of X, all hashing to
    the same bucket and shuffled over the launch.  A re-claim of the bucket
    by X after K's erase restores the word an earlier X insert snapshotted
    (N|OCC|FRESH); that insert must not skip its re-scan.  Every X must end
    up present exactly once with exactly one created flag."""
    import torch

    from paper_1805_03709_b200 import BlockHashSet

    n = 4096
    s = BlockHashSet(n, 1 << 16)
    rng = np.random.default_rng(7)
    P = np.array([73856093, 19349669, 83492791], np.uint64)
    for trial in range(40):
        cand = rng.integers(-(1 << 20), 1 << 20, (8 * n, 3)).astype(np.int32)
        cand = np.unique(cand, axis=0)
        u = cand.astype(np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)
        h = ((u[:, 0] * P[0]) & 0xFFFFFFFF) ^ ((u[:, 1] * P[1]) & 0xFFFFFFFF) ^ ((u[:, 2] * P[2]) & 0xFFFFFFFF)
        b = (h % np.uint64(n)).astype(np.int64)
        order = np.argsort(b, kind="stable")
        bs = b[order]
        first = np.flatnonzero(np.r_[True, bs[1:] != bs[:-1]])
        pairs = [(order[i], order[i + 1]) for i in first if i + 1 < len(bs) and bs[i + 1] == bs[i]]
        K = cand[[p[0] for p in pairs]]
        X = cand[[p[1] for p in pairs]]
        m = len(pairs)
        keys = np.concatenate([K, K, K, X, X, X, X])
        ops = np.concatenate([np.zeros(m), np.full(2 * m, 2), np.zeros(4 * m)]).astype(np.uint8)
        xid = np.concatenate([np.full(3 * m, -1), np.tile(np.arange(m), 4)])
        perm = rng.permutation(len(keys))
        keys, ops, xid = keys[perm], ops[perm], xid[perm]
        res, _ = s.apply(keys, torch.from_numpy(ops))
        s.check_capacity()
        res = res.cpu().numpy()
        created_x = np.bincount(xid[xid >= 0], weights=res[xid >= 0], minlength=m)
        assert np.all(created_x == 1), (trial, np.flatnonzero(created_x != 1)[:8])
        a = s.audit()
        assert a["duplicates"] == 0 and a["unreachable_live"] == 0 and a["free_reachable"] == 0, a
        assert a["free"] + a["reachable_excess"] == s.excess_capacity, a
        found, _ = s.find_keys(X)
        assert bool(found.cpu().numpy().all())
        s.clear()


def test_capacity_exhausted_raises_and_preserves(dev):
    from paper_1805_03709_b200 import BlockHashSet, CapacityExhausted

    s = BlockHashSet(1, 2)
    for key in [(0, 0, 0), (1, 0, 0), (2, 0, 0)]:
        s.insert(key)
    with pytest.raises(CapacityExhausted):
        s.insert((3, 0, 0))
    assert (3, 0, 0) not in s
    assert sorted(s.snapshot_keys()) == [(0, 0, 0), (1, 0, 0), (2, 0, 0)]
    audit_clean(s, 3)


def test_insert_many_exact_prefix_semantics(dev):
    """`for k in keys: insert(k)` semantics on exhaustion: prefix applied."""
    from paper_1805_03709_b200 import BlockHashSet, CapacityExhausted

    keys = [(i, 0, 0) for i in range(40)]
    o = oracle.OracleHashSet(4, 16)
    _, _, fail = o.insert_batch(keys)
    assert fail > 0
    s = BlockHashSet(4, 16)
    with pytest.raises(CapacityExhausted):
        s.insert_many_exact(keys)
    assert sorted(s.snapshot_keys()) == sorted(map(tuple, o.snapshot()[0].tolist()))
    audit_clean(s, o.size())


def test_reference_api_semantics(dev):
    """Ports of tests/test_concurrent_hash.py TestRetrieve/TestInsert/TestRemove/
    TestExtract/TestSnapshot against the GPU classes."""
    from paper_1805_03709_b200 import BlockHashMap, BlockHashSet, hash_key

    s = BlockHashSet(64, 64)
    assert (1, 2, 3) not in s
    s.insert((1, 2, 3))
    assert (1, 2, 3) in s
    assert s.remove((1, 2, 3)) is True and (1, 2, 3) not in s
    assert s.remove((1, 2, 3)) is False

    n = 16
    coll = [(x, 0, 0) for x in range(4000) if hash_key((x, 0, 0), n) == 5][:20]
    s = BlockHashSet(n, 64)
    s.insert(coll[0])
    assert coll[1] not in s
    for k in coll[1:]:
        s.insert(k)
    assert s.remove(coll[0])  # the bucket entry itself
    assert s.remove(coll[7])  # mid-chain
    for i, k in enumerate(coll):
        assert (k in s) == (i not in (0, 7))

    m = BlockHashMap(64, 64)
    m.insert((5, 5, 5), "payload")
    assert m.get((5, 5, 5)) == "payload" and m.get((6, 6, 6)) is None and m.get((6, 6, 6), "d") == "d"
    p1 = m.insert((1, 1, 1), "first")
    p2 = m.insert((1, 1, 1), "second")
    assert p1 == p2 and m.get((1, 1, 1)) == "first"
    m.put((1, 1, 1), "third")
    assert m.get((1, 1, 1)) == "third"
    v, created = m.get_or_create((2, 2, 2), lambda: "made")
    assert (v, created) == ("made", True)
    assert m.get_or_create((2, 2, 2), lambda: "again") == ("made", False)
    assert dict(m.snapshot_items()) == {(5, 5, 5): "payload", (1, 1, 1): "third", (2, 2, 2): "made"}
    assert m.remove((1, 1, 1)) and m.get((1, 1, 1)) is None

    s = BlockHashSet(64, 64)
    keys = [(i, 0, 0) for i in range(5)]
    for k in keys:
        s.insert(k)
    assert sorted(s.extract_batch(10)) == keys and s.approx_size() == 0
    assert s.extract_batch(4) == []
    for i in range(6):
        s.insert((i, 0, 0))
    assert s.extract_matching(10, lambda k: False) == [] and s.approx_size() == 6
    assert len(s.extract_matching(10, lambda k: True)) == 6
    s.insert((-1, 0, 0))
    s.insert((1, 0, 0))
    assert s.extract_matching(10, lambda k: k[0] >= 0) == [(1, 0, 0)]
    assert s.snapshot_keys() == [(-1, 0, 0)]
    assert BlockHashSet(16, 16).snapshot_keys() == []


def test_extract_batch_properties(dev):
    from paper_1805_03709_b200 import BlockHashSet

    s = BlockHashSet(512, 2048)
    keys = {(i, 7, 7) for i in range(1000)}
    s.insert_keys(sorted(keys))
    a = s.extract_batch(600)
    b = s.extract_batch(600)
    assert len(a) == len(set(a)) == 600 and len(b) == len(set(b)) == 400
    assert set(a).isdisjoint(b) and set(a) | set(b) == keys
    assert s.approx_size() == 0
    audit_clean(s, 0)


def test_free_list_conservation_under_churn(dev):
    """tests/test_concurrent_hash.py:366-383 (white-box) via the device audit."""
    from paper_1805_03709_b200 import BlockHashSet

    import random

    s = BlockHashSet(16, 128)
    rng = random.Random(3)
    live = set()
    for _ in range(600):
        k = (rng.randrange(60), 0, 0)
        if rng.random() < 0.5:
            s.insert(k)
            live.add(k)
        else:
            s.remove(k)
            live.discard(k)
    assert set(s.snapshot_keys()) == live
    audit_clean(s, len(live))


def test_whole_set_erase_cycles_keep_free_list_exact(dev):
    """Config 1 as a loop: insert the 100k keys (~20% duplicates), find them
    with 100k absent probes, erase them all -- 60 cycles on one table, audited
    every 10.  Whole-set erases return ~30k excess entries per cycle, which
    fills every free-list stripe exactly (free == excess), and the next
    cycle pops them all again (concurrent_hash.py:72-79, :251-295).  A
    variant that pushed vacated entries from the erase launch itself left
    3-5 freed entries reachable per cycle here (scripts/c1_loop.py)."""
    import torch

    from paper_1805_03709_b200 import BlockHashSet

    keys, absent = workloads.config1_keys()
    dk = torch.from_numpy(keys).to(dev)
    dp = torch.from_numpy(np.concatenate([keys, absent])).to(dev)
    s = BlockHashSet(1 << 17, 1 << 17, device=dev)
    for it in range(60):
        c, _ = s.insert_keys(dk)
        f, _ = s.find_keys(dp)
        e, _ = s.erase_keys(dk)
        assert (int(c.sum()), int(f.sum()), int(e.sum())) == (80_000, 100_000, 80_000), it
        if it % 10 == 9:
            audit_clean(s, 0)
            assert s.audit()["free"] == s.excess_capacity


def test_host_threads_disjoint_key_spaces(dev):
    """tests/test_acceptance.py:229-275 shape, scaled: 8 host threads x 2,000
    per-key ops on disjoint key spaces vs a replayed dict oracle."""
    from paper_1805_03709_b200 import BlockHashMap, BlockHashSet

    for is_map in (False, True):
        s = BlockHashMap(1 << 12, 1 << 12) if is_map else BlockHashSet(1 << 12, 1 << 12)
        logs = {}

        def worker(tid):
            rng = np.random.default_rng(tid)
            ks = rng.integers(0, 300, 2000)
            acts = rng.random(2000)
            log = []
            for i in range(2000):
                key = (tid, int(ks[i]), 0)
                if acts[i] < 0.6:
                    if is_map:
                        s.put(key, (tid, i))
                    else:
                        s.insert(key)
                    log.append((key, (tid, i)))
                else:
                    s.remove(key)
                    log.append((key, None))
            logs[tid] = log

        th = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        expected = {}
        for tid in range(8):
            for key, v in logs[tid]:
                if v is None:
                    expected.pop(key, None)
                else:
                    expected[key] = v
        if is_map:
            assert dict(s.snapshot_items()) == expected
        else:
            assert set(s.snapshot_keys()) == set(expected)
        audit_clean(s, len(expected))


def test_per_key_path_across_recycled_staging(dev):
    """The per-key path (vs_table_single) waits on a completion word in mapped
    pinned memory; pinned blocks are recycled across tables, so a new table
    must never see a previous table's final word as its own completion."""
    from paper_1805_03709_b200 import BlockHashSet

    for rnd in range(4):
        s = BlockHashSet(64, 64)
        for k in range(40 + 10 * rnd):  # seq runs past the previous table's last value
            assert s.insert((k, rnd, 0))
            assert (k, rnd, 0) in s
            assert (k, rnd, 1) not in s
        for k in range(0, 40 + 10 * rnd, 2):
            assert s.remove((k, rnd, 0))
        assert s.approx_size() == (40 + 10 * rnd) // 2
        del s
