"""GPU parity tests of the per-client stream sets and the server update path
against golden sequences recorded from the reference server (tests/golden/).

Bar: each client's pending set bit-exact (sorted); the generation-order
FIFO append order bit-exact (server.py:62-66); extract_ordered results
bit-exact incl. stale-entry skipping (server.py:86-95).
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_streamset_sequences_vs_reference(dev, golden):
    from paper_1805_03709_b200 import StreamSet

    g = json.loads((golden / "stream_seq.json").read_text())
    for name in ("fifo_example", "random"):
        ss = StreamSet(256, 1024)
        for op, arg, want in g[name]:
            if op in ("insert", "remove"):
                assert getattr(ss, op)(tuple(arg)) == want, (op, arg)
            elif op == "insert_many":
                assert ss.insert_many([tuple(a) for a in arg]) == want
            else:
                assert [list(k) for k in ss.extract_ordered(arg)] == want, (op, arg)
    assert sorted(list(k) for k in ss.snapshot()) == g["random_final"]


def test_fifo_keeps_stale_entries_like_the_deque(dev):
    from paper_1805_03709_b200 import StreamSet

    ss = StreamSet(64, 64)
    for k in [(1, 0, 0), (2, 0, 0), (3, 0, 0)]:
        ss.insert(k)
    ss.remove((1, 0, 0))
    ss.insert((4, 0, 0))
    ss.insert((1, 0, 0))
    assert ss.fifo_entries() == [(1, 0, 0), (2, 0, 0), (3, 0, 0), (4, 0, 0), (1, 0, 0)]
    assert ss.extract_ordered(2) == [(1, 0, 0), (2, 0, 0)]
    assert ss.extract_ordered(2) == [(3, 0, 0), (4, 0, 0)]
    assert ss.extract_ordered(2) == []


def test_fifo_growth_and_long_drain(dev):
    from paper_1805_03709_b200 import StreamSet

    rng = np.random.default_rng(2)
    ss = StreamSet(1 << 12, 1 << 12, fifo_capacity=1024)
    o = oracle.OracleStreamSet()
    for step in range(30):
        ks = [tuple(int(v) for v in r) for r in rng.integers(0, 40, (300, 3))]
        assert ss.insert_many(ks) == o.insert_many(ks)
        for k in ks[:20]:
            assert ss.remove(k) == o.remove(k)
        n = int(rng.integers(0, 200))
        assert ss.extract_ordered(n) == o.extract_ordered(n)
    assert ss.extract_ordered(10 ** 6) == o.extract_ordered(10 ** 6)
    assert ss.size() == o.size() == 0


def test_fan_out_40_clients_vs_oracle(dev):
    """insert_many into > 32 clients (two launches) == per-client oracle."""
    from paper_1805_03709_b200 import StreamSet, fan_out, remove_everywhere

    rng = np.random.default_rng(3)
    sets = [StreamSet(1 << 10, 1 << 10) for _ in range(40)]
    oracles = [oracle.OracleStreamSet() for _ in range(40)]
    for c in range(40):  # different pending state per client
        pre = [tuple(int(v) for v in r) for r in rng.integers(0, 12, (c * 3, 3))]
        sets[c].insert_many(pre)
        oracles[c].insert_many(pre)
    for step in range(5):
        upd = [tuple(int(v) for v in r) for r in rng.integers(0, 12, (64, 3))]
        affected = oracle.affected_dedup(upd)
        got = fan_out(sets, affected)
        want = [o.insert_many(affected) for o in oracles]
        assert got == want
        for s, o in zip(sets, oracles):
            assert s.fifo_entries() == list(o.order)
        victims = affected[:5]
        remove_everywhere(sets, victims)
        for o in oracles:
            for v in victims:
                o.remove(v)
    for s, o in zip(sets, oracles):
        assert set(s.snapshot()) == o.set


def test_fan_out_device_count_bound(dev):
    """fan_out(keys, n_dev=k): only the first k keys count (sets, FIFO order,
    created counts), the rest of the buffer is ignored -- the sync-free tick."""
    import torch

    from paper_1805_03709_b200 import StreamSet, fan_out

    rng = np.random.default_rng(11)
    a = [StreamSet(1 << 10, 1 << 10) for _ in range(5)]
    b = [StreamSet(1 << 10, 1 << 10) for _ in range(5)]
    for step in range(4):
        keys = torch.from_numpy(rng.integers(0, 16, (300, 3)).astype(np.int32)).to(dev)
        k = int(rng.integers(0, 301))
        n_dev = torch.tensor([k], dtype=torch.int64, device=dev)
        got = fan_out(a, keys, n_dev=n_dev)
        want = fan_out(b, keys[:k])
        assert got == want, (step, k)
        for x, y in zip(a, b):
            assert x.fifo_entries() == y.fifo_entries()
            assert set(x.snapshot()) == set(y.snapshot())


@pytest.mark.parametrize("u,span", [(700, 5), (1, 5), (1024, 5), (1024, 1000), (1025, 5), (3000, 40)])
def test_affected_dedup_order(dev, u, span):
    """u <= 1024 runs the one-CTA shared-memory dedup, larger batches the
    scratch-table path; both must give the first-occurrence order."""
    import torch

    from paper_1805_03709_b200 import BlockHashSet, _lib

    rng = np.random.default_rng(9 + u)
    upd = rng.integers(-span, span, (u, 3)).astype(np.int32)
    scratch = BlockHashSet(1 << 14, 1 << 14)
    out = torch.empty((8 * u, 3), dtype=torch.int32, device=dev)
    n = torch.empty(1, dtype=torch.int64, device=dev)
    k = torch.from_numpy(upd).to(dev)
    for _ in range(2):  # the scratch path must also work on a reused scratch set
        _lib.check(_lib.load().vs_affected_dedup(scratch.handle, _lib.ptr(k), u, _lib.ptr(out), _lib.ptr(n),
                                                 _lib.stream_of(dev)))
        got = [tuple(r) for r in out[: int(n.item())].cpu().tolist()]
        assert got == oracle.affected_dedup(upd.tolist())


@pytest.mark.parametrize("sync", [True, False])
def test_server_core_replays_reference_server(dev, golden, sync):
    """Server.on_tsdf_batch / on_reset_blocks / fresh attach, replayed on the
    GPU core with the reference's exact TSDF bytes (server_blocks.npz);
    sync=False runs each batch as ONE vs_server_tick call."""
    from paper_1805_03709_b200 import GpuServerCore

    g = json.loads((golden / "server_seq.json").read_text())
    d = np.load(golden / "server_blocks.npz")
    core = GpuServerCore(1 << 12, 1 << 12, stream_buckets=1 << 10, stream_excess=1 << 10)
    clients = [core.attach(bytes([i]) * 16) for i in range(3)]
    for step, entry in enumerate(g["steps"]):
        sel = d["step"] == step
        keys = d["keys"][sel]
        assert keys.tolist() == entry["updated"]
        before = [len(c.fifo_entries()) for c in clients]
        core.on_tsdf_batch(keys, d["blocks"][sel], sync=sync)
        for c, cl in enumerate(clients):
            assert [list(k) for k in cl.fifo_entries()[before[c]:]] == entry["appended"][c]
            assert sorted(list(k) for k in cl.snapshot()) == entry["pending"][c]
        if "pending_after_extract_c1" in entry:
            keep = {tuple(k) for k in entry["pending_after_extract_c1"]}
            drop = [k for k in clients[1].snapshot() if k not in keep]
            clients[1].remove_many(drop)  # adopt the reference's random subset
        if "reset" in entry:
            core.on_reset_blocks([tuple(v) for v in entry["reset"]])
            for c, cl in enumerate(clients):
                assert sorted(list(k) for k in cl.snapshot()) == entry["pending_after_reset"][c]
    keys, _ = core.mc_map.snapshot_tensor()
    got = sorted(tuple(k) for k in keys.cpu().tolist())
    assert [list(k) for k in got] == g["mc_keys"]
    for k in got:
        digest = hashlib.sha256(core.mc_payload(k)).hexdigest()
        assert digest == g["mc_digest"][",".join(map(str, k))], k
    fresh = core.attach(b"\x09" * 16)
    assert sorted(list(k) for k in fresh.snapshot()) == g["fresh_pending"]
    # a returning client keeps its set (server.py:225-239)
    assert core.attach(bytes([0]) * 16) is clients[0]


def test_config4_tick_loop_vs_oracle(dev):
    """Config-4 shape at reduced scale: fresh fills, update ticks fanned out to
    every client, random extraction, fresh reconnect and resets -- each
    client's pending set and FIFO stay equal to the reference-semantics oracle."""
    import torch

    from paper_1805_03709_b200 import StreamSet, fan_out, remove_everywhere, workloads

    scene = workloads.room_block_keys()
    scene = scene[(scene[:, 0] <= -170) & (scene[:, 2] <= -170)]
    scene_t = [tuple(k) for k in scene.tolist()]
    rng = np.random.default_rng(8)
    C = 4
    gpu = [StreamSet(1 << 14, 1 << 14, fifo_capacity=1 << 12) for _ in range(C)]
    ref = [oracle.OracleStreamSet() for _ in range(C)]
    assert fan_out(gpu, scene) == [len(scene)] * C
    for r in ref:
        r.insert_many(scene_t)
    for t in range(30):
        upd = [scene_t[i] for i in rng.integers(0, len(scene_t), 64)]
        aff = oracle.affected_dedup(upd)
        assert fan_out(gpu, aff) == [r.insert_many(aff) for r in ref]
        for g, r in zip(gpu, ref):
            got = g.extract_random(50)
            assert len(got) == len(set(got)) == min(50, r.size())
            for k in got:
                assert r.remove(k)  # the GPU's random subset, adopted by the oracle
        if t % 10 == 9:
            v = t // 10 % C
            gpu[v].clear()
            ref[v] = oracle.OracleStreamSet()
            fan_out([gpu[v]], scene)
            ref[v].insert_many(scene_t)
            reset = [scene_t[i] for i in rng.integers(0, len(scene_t), 32)]
            remove_everywhere(gpu, reset)
            for r in ref:
                for k in reset:
                    r.remove(k)
    for g, r in zip(gpu, ref):
        assert set(g.snapshot()) == r.set
        assert g.fifo_entries() == list(r.order)  # stale entries included
        assert g.extract_ordered(10 ** 6) == r.extract_ordered(10 ** 6)


def test_stream_tick_fused_vs_oracle(dev):
    """vs_stream_tick (dedup + fan-out + extraction in ONE launch): the
    affected list equals the reference's dict-order dedup, every client's
    pending set and FIFO (stale entries included) stay equal to the oracle
    through reconnects and resets, extraction counts = min(max_n, size),
    tables audit clean (the extraction recycles in the same launch)."""
    import torch

    from paper_1805_03709_b200 import StreamSet, fan_out, remove_everywhere, stream_tick, workloads

    scene = workloads.room_block_keys()
    scene = scene[(scene[:, 0] <= -170) & (scene[:, 2] <= -170)]
    scene_t = [tuple(k) for k in scene.tolist()]
    rng = np.random.default_rng(10)
    C, X = 5, 60
    # 28k structured keys collide heavily under the normative hash: 2^15 + 2^15
    # entries keep the excess region clear of exhaustion (checked below)
    gpu = [StreamSet(1 << 15, 1 << 15, fifo_capacity=1 << 12) for _ in range(C)]
    ref = [oracle.OracleStreamSet() for _ in range(C)]
    fan_out(gpu, scene)
    for r in ref:
        r.insert_many(scene_t)
    for t in range(30):
        U = int(rng.integers(1, 513)) if t % 3 else 512
        idx = rng.integers(0, len(scene_t), U)
        if t == 4:  # colliding updates: many duplicates among the expanded keys
            idx = np.repeat(idx[:8], U // 8 + 1)[:U]
        upd = [scene_t[i] for i in idx]
        aff_want = oracle.affected_dedup(upd)
        aff, na, keys, n = stream_tick(gpu, torch.from_numpy(scene[idx]).to(dev), X, seeds=[t * 7 + c for c in range(C)])
        assert int(na.item()) == len(aff_want)
        assert [tuple(k) for k in aff[: len(aff_want)].cpu().tolist()] == aff_want
        for c, r in enumerate(ref):
            r.insert_many(aff_want)
            got = [tuple(k) for k in keys[c, : int(n[c])].cpu().tolist()]
            assert len(got) == len(set(got)) == min(X, r.size())
            for k in got:
                assert r.remove(k)
        if t % 10 == 9:
            v = t // 10 % C
            gpu[v].clear()
            ref[v] = oracle.OracleStreamSet()
            fan_out([gpu[v]], scene)
            ref[v].insert_many(scene_t)
            reset = [scene_t[i] for i in rng.integers(0, len(scene_t), 32)]
            remove_everywhere(gpu, reset)
            for r in ref:
                for k in reset:
                    r.remove(k)
    for g, r in zip(gpu, ref):
        g._set.check_capacity()
        assert g.size() == len(r.set)
        assert set(g.snapshot()) == r.set
        assert g.fifo_entries() == list(r.order)
        a = g._set.audit()
        assert a["duplicates"] == 0 and a["unreachable_live"] == 0 and a["free_reachable"] == 0
        assert a["free"] + a["reachable_excess"] == g._set.excess_capacity


def test_stream_tick_edges(dev):
    """vs_stream_tick with a single updated key and no extraction, with
    max_n larger than every set, and the argument checks."""
    import torch

    from paper_1805_03709_b200 import StreamSet, stream_tick

    sets = [StreamSet(1 << 10, 1 << 10) for _ in range(3)]
    aff, na, keys, n = stream_tick(sets, torch.tensor([[5, 6, 7]], dtype=torch.int32, device=dev), 0, seeds=[1, 2, 3])
    want = oracle.affected_dedup([(5, 6, 7)])
    assert int(na.item()) == 8 and [tuple(k) for k in aff.cpu().tolist()] == want
    assert n.cpu().tolist() == [0, 0, 0]
    for st in sets:
        assert sorted(st.snapshot()) == sorted(want) and st.fifo_entries() == want
    aff, na, keys, n = stream_tick(sets, torch.tensor([[5, 6, 7]], dtype=torch.int32, device=dev), 100, seeds=[4, 5, 6])
    assert n.cpu().tolist() == [8, 8, 8]  # nothing new was created: all 8 pending keys come out
    for c, st in enumerate(sets):
        assert sorted(tuple(k) for k in keys[c, :8].cpu().tolist()) == sorted(want)
        assert st.size() == 0
    with pytest.raises(ValueError):
        stream_tick(sets, torch.zeros((513, 3), dtype=torch.int32, device=dev), 1)


def test_stream_set_grows_past_its_capacity(dev):
    """The reference caps a client's set at 2^16 + 2^16 entries and raises
    CapacityExhausted on larger models (server.py:242-243); our StreamSet
    grows instead: every key pending and queued exactly once.  (Keys whose
    insert found the old table full are queued after the rest of that call:
    there is no reference order for a call the reference would have failed.)
    A set that did not overflow keeps the exact generation order."""
    from paper_1805_03709_b200 import StreamSet, fan_out

    rng = np.random.default_rng(4)
    keys = [tuple(int(v) for v in r) for r in np.unique(rng.integers(-10**6, 10**6, (6000, 3)), axis=0)]
    ref = oracle.OracleStreamSet()
    small = StreamSet(1 << 6, 1 << 6, fifo_capacity=1 << 10)
    other = StreamSet(1 << 14, 1 << 14)
    half = len(keys) // 2
    assert fan_out([small, other], keys[:half]) == [half, half]
    assert small.insert_many(keys) == len(keys) - half
    ref.insert_many(keys)
    assert small.size() == len(keys) and set(small.snapshot()) == ref.set
    assert sorted(small.fifo_entries()) == sorted(ref.order)
    got = small.extract_ordered(100)
    assert len(got) == 100 and set(got) <= ref.set
    assert other.fifo_entries() == keys[:half]
    a = small._set.audit()
    assert a["duplicates"] == 0 and a["unreachable_live"] == 0


def test_extract_random_many_properties(dev):
    """Windowed multi-client extraction: distinct keys, subset of the set,
    count = min(max_n, size), post-set = pre-set minus returned, rotation
    start honoured (positions ascending from the start, wrapping)."""
    from paper_1805_03709_b200 import StreamSet, extract_random_many

    rng = np.random.default_rng(5)
    sets = [StreamSet(1 << 12, 1 << 12) for _ in range(5)]
    pre = []
    for i, s in enumerate(sets):
        ks = {tuple(int(v) for v in r) for r in rng.integers(-50, 50, (200 * (i + 1), 3))}
        s.insert_many(sorted(ks))
        pre.append(ks)
    keys, n = extract_random_many(sets, 300, seeds=[1, 2, 3, 4, 5])
    for i, s in enumerate(sets):
        got = [tuple(k) for k in keys[i, : int(n[i])].cpu().tolist()]
        assert len(got) == len(set(got)) == min(300, len(pre[i]))
        assert set(got) <= pre[i]
        assert set(s.snapshot()) == pre[i] - set(got)
        a = s._set.audit()
        assert a["duplicates"] == 0 and a["free"] + a["reachable_excess"] == s._set.excess_capacity


def test_visible_first_predicate_bit_exact_with_reference(dev, golden):
    """Device frustum-AABB decisions == Server._visibility_predicate (recorded
    from the reference after the wire's float32 round trip)."""
    from paper_1805_03709_b200 import BlockHashSet

    d = np.load(golden / "visibility.npz")
    for t in range(d["keys"].shape[0]):
        keys = d["keys"][t]
        uniq, first = np.unique(keys, axis=0, return_index=True)
        vis = d["visible"][t][first]
        s = BlockHashSet(1 << 15, 1 << 15)
        s.insert_keys(uniq)
        got = s.extract_visible(len(uniq), d["planes"][t], float(d["margin"][t]), float(d["block"][t]))
        want = {tuple(k) for k, v in zip(uniq.tolist(), vis) if v}
        assert set(got) == want and len(got) == len(want), t
        assert s.approx_size() == len(uniq) - len(want)
        # bounded request: max_n visible keys, all visible, distinct
        s2 = BlockHashSet(1 << 15, 1 << 15)
        s2.insert_keys(uniq)
        some = s2.extract_visible(7, d["planes"][t], float(d["margin"][t]), float(d["block"][t]))
        assert len(some) == min(7, len(want)) and set(some) <= want


def test_block_request_strategies_and_mc_batch_payload(dev, golden):
    """Server.on_block_request (server.py:334-363) on the GPU core: strategies
    and the MC_BATCH payload layout (wire.py:292-299)."""
    import struct

    from paper_1805_03709_b200 import GpuServerCore

    d = np.load(golden / "server_blocks.npz")
    core = GpuServerCore(1 << 12, 1 << 12, stream_buckets=1 << 10, stream_excess=1 << 10)
    cid = b"c" * 16
    st = core.attach(cid)
    core.on_tsdf_batch(d["keys"], d["blocks"])
    pending = set(st.snapshot())
    fifo = [k for k in st.fifo_entries()]
    keys, payload = core.on_block_request(cid, 10, 0)  # generation order
    assert keys == fifo[:10]
    n = struct.unpack_from("<I", payload, 0)[0]
    assert n == len(keys) and len(payload) == 4 + 2060 * n
    for i, k in enumerate(keys):
        off = 4 + 2060 * i
        assert struct.unpack_from("<3i", payload, off) == k
        assert payload[off + 12: off + 2060] == core.mc_payload(k)
    keys2, _ = core.on_block_request(cid, 25, 2)  # random
    assert len(keys2) == 25 and set(keys2) <= pending - set(keys)
    v = np.load(golden / "visibility.npz")
    keys3, payload3 = core.on_block_request(cid, 30, 1, v["planes"][0], float(v["margin"][0]), float(v["block"][0]))
    assert len(keys3) == 30 and len(set(keys3)) == 30  # visible first, topped up
    assert set(st.snapshot()) == pending - set(keys) - set(keys2) - set(keys3)


def test_tsdf_ingest_latest_write_wins(dev):
    """tsdf_map.put semantics (server.py:300-303, tests/test_server.py
    test_latest_write_wins) incl. duplicate keys inside one batch."""
    from paper_1805_03709_b200 import GpuServerCore

    rng = np.random.default_rng(1)
    core = GpuServerCore(1 << 10, 1 << 10, stream_buckets=1 << 9, stream_excess=1 << 9)
    keys = np.array([[2, 2, 2], [3, 2, 2], [2, 2, 2], [4, 4, 4], [2, 2, 2]], np.int32)
    rows = rng.integers(0, 256, (5, 6144), dtype=np.uint8)
    core.on_tsdf_batch(keys, rows)
    assert core.tsdf_payload((2, 2, 2)) == rows[4].tobytes()
    assert core.tsdf_payload((3, 2, 2)) == rows[1].tobytes()
    rows2 = rng.integers(0, 256, (1, 6144), dtype=np.uint8)
    core.on_tsdf_batch(keys[:1], rows2)
    assert core.tsdf_payload((2, 2, 2)) == rows2[0].tobytes()
    assert core.tsdf_map.approx_size() == 3


def test_server_core_concurrent_session_threads(dev):
    """The reference Server calls on_tsdf_batch and on_block_request from
    different session threads (transport.py:157-160).  Ticks on one thread
    and block requests of two clients on two others, each thread on its own
    CUDA stream: no exception, every table passes its audit, no capacity
    error, and what each client received plus what it still holds is exactly
    the set of MC keys the ticks produced (nothing lost; a key updated again
    after its delivery is pending again, as in the reference)."""
    import threading

    import torch

    from paper_1805_03709_b200 import GpuServerCore, workloads

    scene = workloads.room_block_keys()[:40_000]
    core = GpuServerCore(1 << 17, 1 << 17, stream_buckets=1 << 17, stream_excess=1 << 17, max_batch=1 << 10,
                         device=dev)
    ids = [bytes([c]) * 16 for c in range(2)]
    for cid in ids:
        core.attach(cid)
    rng = np.random.default_rng(3)
    upd = [scene[rng.integers(0, len(scene), 512)] for _ in range(24)]
    rows = [workloads.room_tsdf_rows(torch.from_numpy(u).to(dev)) for u in upd]
    got = {cid: [] for cid in ids}
    errors = []

    def ticks():
        try:
            with torch.cuda.stream(torch.cuda.Stream(dev)):
                for u, r in zip(upd, rows):
                    core.on_tsdf_batch(u, r, sync=False)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    def requests(cid, strategy):
        try:
            with torch.cuda.stream(torch.cuda.Stream(dev)):
                for _ in range(40):
                    keys, _ = core.on_block_request(cid, 256, strategy)
                    got[cid].extend(keys)
        except Exception as e:  # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=ticks)] + [threading.Thread(target=requests, args=(cid, s))
                                             for cid, s in zip(ids, (0, 2))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors
    core.check()
    for t in [core.tsdf_map, core.mc_map] + [core.sessions[cid]["stream"]._set for cid in ids]:
        a = t.audit()
        assert a["duplicates"] == 0 and a["unreachable_live"] == 0 and a["free_reachable"] == 0, a
    produced = {tuple(k) for k in core.mc_map.snapshot_keys()}
    for cid in ids:
        st = core.sessions[cid]["stream"]
        sent = {tuple(k) for k in got[cid]}
        pending = {tuple(k) for k in st.snapshot()}
        assert sent and pending | sent == produced
