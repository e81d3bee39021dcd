"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (the reference exists only there):

    cd /tmp && PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python /root/repo/tests/golden/gen_golden.py

It imports the unmodified reference package ``voxelstream`` (read-only mount)
and records its outputs on seeded inputs; the committed fixtures then pin the
oracle (oracle/) and, through it, the CUDA path, on the GPU box where the
reference is absent.  Nothing in the product or the GPU tests reads
/root/reference at run time.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import os
import pathlib
import random
import sys

import numpy as np

OUT = pathlib.Path(__file__).resolve().parent
REF = pathlib.Path("/root/reference/pkg/src")
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

from voxelstream import concurrent_hash as ch  # noqa: E402
from voxelstream import mc_encoding as mce  # noqa: E402
from voxelstream import server as srv_mod  # noqa: E402
from voxelstream import wire  # noqa: E402
from voxelstream.voxel_model import TsdfBlock  # noqa: E402

sys.path.insert(0, str(OUT.parent.parent))
from paper_1805_03709_b200 import workloads  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --------------------------------------------------------------- hash KATs

def gen_hash_kat() -> None:
    rng = random.Random(7)
    cases = [((0, 0, 0), 1 << 20), ((1, 0, 0), 1 << 30), ((1, 2, 3), 1 << 20), ((-1, 0, 0), 97),
             ((-1, -1, -1), 1 << 20), ((2**31 - 1, -2**31, 7), 1000003), ((123, -456, 789), (1 << 20) + 7)]
    for _ in range(300):
        key = tuple(rng.randint(-(2**31), 2**31 - 1) for _ in range(3))
        n = rng.choice([1, 2, 97, 1023, 1 << 17, 7142858, (1 << 31) - 1, 1 << 20])
        cases.append((key, n))
    out = [{"key": list(k), "n": n, "bucket": ch.hash_key(k, n)} for k, n in cases]
    (OUT / "hash_kat.json").write_text(json.dumps(out))


# ------------------------------------------------------- hash op sequences

def record_ops(s, ops_keys):
    """Apply (op, key) on a reference set; op 0 insert, 1 find, 2 erase.
    Returns result flags and positions exactly as the reference computes them."""
    res, pos = [], []
    for op, k in ops_keys:
        if op == 0:
            p, c = s._insert_pos(k)
            res.append(int(c)); pos.append(p)
        elif op == 1:
            p = s._find(k)
            res.append(int(p is not None)); pos.append(-1 if p is None else p)
        else:
            p = s._find(k)
            r = s.remove(k)
            res.append(int(r)); pos.append(-1 if not r else p)
    return res, pos


def snapshot_state(s):
    keys = []
    pos = []
    for e in np.flatnonzero(s._occ):
        keys.append(list(s._keys[e])); pos.append(int(e))
    return {"keys": keys, "pos": pos, "free": list(s.free_stack._slots),
            "next": [int(v) for v in s._next]}


def gen_hash_seq() -> None:
    scenarios = {}
    # (a) the reference's randomized sequence shape (tests/test_concurrent_hash.py:273-285)
    #     with finds mixed in, on a small table that forces long chains
    rng = random.Random(42)
    ops = []
    for _ in range(20000):
        key = (rng.randrange(40), rng.randrange(5), 0)
        r = rng.random()
        ops.append((0 if r < 0.5 else (1 if r < 0.7 else 2), key))
    s = ch.BlockHashSet(16, 512)
    res, pos = record_ops(s, ops)
    scenarios["rand42"] = {"n": 16, "excess": 512, "ops": [o for o, _ in ops], "keys": [list(k) for _, k in ops],
                           "res": res, "pos": pos, "final": snapshot_state(s)}
    # (b) one colliding chain: insert 20, remove the bucket entry and a middle one, reinsert
    n = 16
    coll = []
    x = 0
    while len(coll) < 24:
        if ch.hash_key((x, 0, 0), n) == 3:
            coll.append((x, 0, 0))
        x += 1
    ops = [(0, k) for k in coll[:20]] + [(2, coll[0]), (2, coll[7]), (1, coll[8]), (1, coll[7])]
    ops += [(0, k) for k in coll[20:]] + [(0, coll[7]), (2, coll[19]), (1, coll[19]), (0, coll[0])]
    s = ch.BlockHashSet(n, 64)
    res, pos = record_ops(s, ops)
    scenarios["chain"] = {"n": n, "excess": 64, "ops": [o for o, _ in ops], "keys": [list(k) for _, k in ops],
                          "res": res, "pos": pos, "final": snapshot_state(s)}
    # (c) capacity exhaustion (tests/test_concurrent_hash.py:129-136)
    s = ch.BlockHashSet(1, 2)
    for k in [(0, 0, 0), (1, 0, 0), (2, 0, 0)]:
        s.insert(k)
    try:
        s.insert((3, 0, 0))
        raised = False
    except ch.CapacityExhausted:
        raised = True
    scenarios["capacity"] = {"n": 1, "excess": 2, "raised": raised, "final": snapshot_state(s)}
    (OUT / "hash_seq.json").write_text(json.dumps(scenarios))


def gen_config1() -> None:
    """Config 1 (BASELINE.json configs[0]) hash half, recorded from the reference:
    digests only (the generator in workloads.py rebuilds the inputs)."""
    keys, absent = workloads.config1_keys()
    s = ch.BlockHashSet(1 << 17, 1 << 17)
    created, ins_pos = [], []
    for k in map(tuple, keys.tolist()):
        p, c = s._insert_pos(k)
        created.append(c); ins_pos.append(p)
    probe = np.concatenate([keys, absent])
    found, find_pos = [], []
    for k in map(tuple, probe.tolist()):
        p = s._find(k)
        found.append(p is not None); find_pos.append(-1 if p is None else p)
    snap = np.asarray(s.snapshot_keys(), dtype=np.int32)
    erased = []
    for k in map(tuple, keys.tolist()):
        erased.append(s.remove(k))
    out = {
        "keys_sha": sha(keys), "absent_sha": sha(absent),
        "created_sha": sha(np.asarray(created, np.uint8)), "created_sum": int(sum(created)),
        "insert_pos_sha": sha(np.asarray(ins_pos, np.int32)),
        "found_sha": sha(np.asarray(found, np.uint8)), "found_sum": int(sum(found)),
        "find_pos_sha": sha(np.asarray(find_pos, np.int32)),
        "erased_sha": sha(np.asarray(erased, np.uint8)), "erased_sum": int(sum(erased)),
        "snapshot_sorted_sha": sha(snap[np.lexsort(snap.T[::-1])]),
        "final_size": s.approx_size(),
    }
    (OUT / "config1_hash.json").write_text(json.dumps(out, indent=1))


# ------------------------------------------------------------------- MC

def _block(key, tsdf, weight, color):
    b = TsdfBlock(key)
    b.tsdf = tsdf.astype(np.float32)
    b.weight = weight.astype(np.float32)
    b.color = color.astype(np.uint8)
    return b


def gen_mc_random() -> None:
    rng = np.random.default_rng(11)
    tkeys = list(itertools.product(range(3), repeat=3))
    T = len(tkeys)
    tsdf = rng.uniform(-1, 1, (T, 512)).astype(np.float32)
    weight = (rng.random((T, 512)) > 0.15).astype(np.float32) * rng.uniform(0.5, 128, (T, 512)).astype(np.float32)
    color = rng.integers(0, 256, (T, 512, 3)).astype(np.uint8)
    # IEEE edge cases sprinkled in
    specials_t = np.array([np.nan, -0.0, 0.0, -1e-45, 1e-45, np.inf, -np.inf, -1e-38, 1e-38], np.float32)
    specials_w = np.array([np.nan, -1.0, 1e-45, np.inf, -0.0, 0.0, -np.inf], np.float32)
    for _ in range(400):
        tsdf[rng.integers(T), rng.integers(512)] = specials_t[rng.integers(len(specials_t))]
        weight[rng.integers(T), rng.integers(512)] = specials_w[rng.integers(len(specials_w))]
    blocks = {k: _block(k, tsdf[i], weight[i], color[i]) for i, k in enumerate(tkeys)}
    mkeys = sorted({a for k in tkeys for a in mce.affected_mc_blocks(k)} | set(tkeys))
    mc = np.stack([np.frombuffer(mce.recompute_mc_block(k, blocks.get).to_bytes(), np.uint8) for k in mkeys])
    np.savez_compressed(OUT / "mc_random.npz", tsdf_keys=np.asarray(tkeys, np.int32), tsdf=tsdf, weight=weight,
                        color=color, mc_keys=np.asarray(mkeys, np.int32), mc=mc)


def gen_mc_edge() -> None:
    """8 neighbours tsdf 0.5/weight 1, centre voxel 1 at
    -0.5; vary voxel 0.  Recorded from the reference vectorised path."""
    cases = [(-0.5, 1.0), (-0.0, 1.0), (float("nan"), 1.0), (-0.5, float("nan")), (-0.5, -1.0),
             (-0.5, float("inf")), (-1e-45, 1.0), (-0.5, 1e-45), (float("-inf"), 1.0), (1e-45, 1.0)]
    out = []
    for t0, w0 in cases:
        blocks = {}
        for k in itertools.product((0, 1), repeat=3):
            b = _block(k, np.full(512, 0.5), np.ones(512), np.full((512, 3), 7))
            blocks[k] = b
        c = blocks[(0, 0, 0)]
        c.tsdf[1] = -0.5
        c.tsdf[0] = np.float32(t0)
        c.weight[0] = np.float32(w0)
        mc = mce.recompute_mc_block((0, 0, 0), blocks.get)
        out.append({"tsdf0": repr(t0), "weight0": repr(w0), "index0": int(mc.index[0]),
                    "mc_sha": hashlib.sha256(mc.to_bytes()).hexdigest()})
    (OUT / "mc_edge.json").write_text(json.dumps(out, indent=1))


def gen_mc_sphere() -> None:
    """The fused-sphere model behind manifest.json's model_sha256
    (fixtures.build_model_blocks, fixtures.py:28-41): store its TSDF blocks."""
    from voxelstream.dataset import SphereScene, default_intrinsics, synthetic_frames
    from voxelstream.voxel_model import FusionConfig, VoxelModel

    scene = SphereScene(radius=0.4, orbit_radius=1.4)
    intr = default_intrinsics(80, 60)
    model = VoxelModel(FusionConfig(voxel_size=0.01, truncation=0.06), bucket_count=1 << 13,
                       excess_capacity=1 << 13)
    for frame in synthetic_frames(scene, intr, 8):
        model.allocate_blocks(frame.depth, frame.pose, intr)
        model.integrate_frame(frame.depth, frame.color, frame.pose, intr)
    keys = sorted(model.keys())
    blocks = [model.get_block(k) for k in keys]
    tsdf = np.stack([b.tsdf for b in blocks]).astype(np.float32)
    weight = np.stack([b.weight for b in blocks]).astype(np.float32)
    color = np.stack([b.color for b in blocks]).astype(np.uint8)
    digest = hashlib.sha256(b"".join(mce.recompute_mc_block(k, model.get_block).to_bytes() for k in keys)).hexdigest()
    manifest = json.loads((REF.parent / "fixtures" / "protocol" / "manifest.json").read_text())
    assert digest == manifest["model_sha256"], "reference fused sphere no longer reproduces the manifest digest"
    np.savez_compressed(OUT / "mc_sphere.npz", keys=np.asarray(keys, np.int32), tsdf=tsdf, weight=weight,
                        color=color)
    (OUT / "mc_sphere.json").write_text(json.dumps({"model_sha256": digest, "model_blocks": len(keys)}))


# ------------------------------------------------------------ stream sets

def gen_stream() -> None:
    out = {}
    # FIFO semantics incl. stale entries (SURVEY A10 example)
    ss = srv_mod.StreamSet(64, 64)
    log = []
    for op, arg in [("insert", (1, 0, 0)), ("insert", (2, 0, 0)), ("insert", (3, 0, 0)), ("remove", (1, 0, 0)),
                    ("insert", (4, 0, 0)), ("insert", (1, 0, 0)), ("extract_ordered", 2), ("extract_ordered", 2),
                    ("extract_ordered", 2)]:
        r = getattr(ss, op)(arg)
        log.append([op, list(arg) if isinstance(arg, tuple) else arg,
                    [list(k) for k in r] if isinstance(r, list) else r])
    out["fifo_example"] = log
    # random op sequence
    rng = random.Random(5)
    ss = srv_mod.StreamSet(256, 1024)
    log = []
    for _ in range(3000):
        r = rng.random()
        if r < 0.45:
            k = (rng.randrange(60), rng.randrange(3), 1)
            log.append(["insert", list(k), ss.insert(k)])
        elif r < 0.6:
            ks = [(rng.randrange(60), rng.randrange(3), 1) for _ in range(rng.randrange(1, 9))]
            log.append(["insert_many", [list(k) for k in ks], ss.insert_many(ks)])
        elif r < 0.8:
            k = (rng.randrange(60), rng.randrange(3), 1)
            log.append(["remove", list(k), ss.remove(k)])
        else:
            n = rng.randrange(0, 7)
            log.append(["extract_ordered", n, [list(k) for k in ss.extract_ordered(n)]])
    out["random"] = log
    out["random_final"] = sorted(list(k) for k in ss.snapshot())
    (OUT / "stream_seq.json").write_text(json.dumps(out))


class _Conn:
    def __init__(self):
        self.sent = []
        self.bytes_sent = 0
        self.bytes_received = 0

    def send(self, msg, codec=0):
        self.sent.append(msg)

    def close(self):
        pass


def gen_server() -> None:
    """Server.on_tsdf_batch fan-out + reset + fresh attach, recorded per client."""
    random.seed(0)  # extract_batch draws its start with random.randrange
    s = srv_mod.Server(srv_mod.ServerConfig(buckets=1 << 12, excess=1 << 12, voxel_size=0.01))
    sessions = []
    for i in range(3):
        sess = s._attach_session(wire.Hello(wire.Role.EXPLORATION, bytes([i]) * 16, 0.01), _Conn())
        sessions.append(sess)
    rng = np.random.default_rng(4)
    steps = []
    raw_keys, raw_blocks, raw_step = [], [], []
    for step in range(6):
        u = int(rng.integers(1, 12))
        upd = [tuple(int(v) for v in rng.integers(-3, 4, 3)) for _ in range(u)]
        blocks = []
        for k in upd:
            b = TsdfBlock(k)
            b.tsdf = rng.uniform(-1, 1, 512).astype(np.float32)
            b.weight = (rng.random(512) > 0.1).astype(np.float32)
            b.color = rng.integers(0, 256, (512, 3)).astype(np.uint8)
            blocks.append((k, b.to_bytes()))
            raw_keys.append(k)
            raw_blocks.append(np.frombuffer(b.to_bytes(), np.uint8))
            raw_step.append(step)
        before = [list(ss.stream._order) for ss in sessions]
        s.on_tsdf_batch(wire.TsdfBatch(blocks))
        entry = {"updated": [list(k) for k in upd],
                 "tsdf_sha": [hashlib.sha256(raw).hexdigest() for _, raw in blocks],
                 "appended": [[list(k) for k in list(ss.stream._order)[len(b):]] for ss, b in zip(sessions, before)],
                 "pending": [sorted(list(k) for k in ss.stream.snapshot()) for ss in sessions]}
        if step == 2:
            sessions[1].stream.extract_random(5)
            entry["pending_after_extract_c1"] = sorted(list(k) for k in sessions[1].stream.snapshot())
        if step == 4:
            victims = [list(k) for k in upd[:2]]
            s.on_reset_blocks([tuple(v) for v in victims])
            entry["reset"] = victims
            entry["pending_after_reset"] = [sorted(list(k) for k in ss.stream.snapshot()) for ss in sessions]
        steps.append(entry)
    mc_keys = sorted(list(k) for k in s.mc_map.snapshot_keys())
    mc_digest = {",".join(map(str, k)): hashlib.sha256(s.mc_map.get(tuple(k))).hexdigest() for k in mc_keys}
    fresh = s._attach_session(wire.Hello(wire.Role.EXPLORATION, b"\x09" * 16, 0.01), _Conn())
    out = {"steps": steps, "mc_keys": mc_keys, "mc_digest": mc_digest,
           "fresh_pending": sorted(list(k) for k in fresh.stream.snapshot())}
    # the TSDF payloads themselves, so the GPU test replays the exact bytes
    np.savez_compressed(OUT / "server_blocks.npz", keys=np.asarray(raw_keys, np.int32),
                        blocks=np.stack(raw_blocks), step=np.asarray(raw_step, np.int32))
    (OUT / "server_seq.json").write_text(json.dumps(out))


def gen_visibility() -> None:
    """Server._visibility_predicate (server.py:365-387) decisions for block
    keys around four camera poses, after the wire's float32 round trip."""
    from voxelstream.geometry import CameraIntrinsics, Frustum, Pose

    s = srv_mod.Server(srv_mod.ServerConfig(buckets=1 << 10, excess=1 << 10, voxel_size=0.01))
    rng = np.random.default_rng(12)
    planes, margins, blocks, keys_all, vis_all, poses, intrs = [], [], [], [], [], [], []
    for trial in range(4):
        eye = rng.uniform(-1, 1, 3)
        pose = Pose.look_at(eye, eye + rng.normal(size=3))
        pose_f = tuple(float(v) for v in np.concatenate([pose.rotation.reshape(-1), pose.translation]))
        intr = (float(rng.uniform(30, 80)), float(rng.uniform(30, 80)), 40.0, 30.0, 0.05, float(rng.uniform(1, 3)))
        req = wire.decode_message(wire.encode_message(
            wire.BlockRequest(64, wire.Strategy.VISIBLE_FIRST, pose_f, intr), 0))
        pred = s._visibility_predicate(req)
        block = 8 * 0.01  # BLOCK_EDGE * voxel_size (server.py:366-367)
        fx, fy, cx, cy, near, far = req.intrinsics
        fr = Frustum(Pose.from_floats(req.pose), CameraIntrinsics(fx=fx, fy=fy, cx=cx, cy=cy, width=int(2 * cx) or 640,
                                                                   height=int(2 * cy) or 480),
                     near=max(near, 1e-3), far=far, margin=block)
        c = np.floor(eye / block).astype(np.int64)
        keys = (c + rng.integers(-45, 46, (20000, 3))).astype(np.int32)
        vis = np.array([pred(tuple(int(v) for v in k)) for k in keys], dtype=bool)
        planes.append(fr._planes)
        margins.append(fr.margin)
        blocks.append(block)
        keys_all.append(keys)
        vis_all.append(vis)
        poses.append(req.pose)
        intrs.append(req.intrinsics)
    np.savez_compressed(OUT / "visibility.npz", planes=np.stack(planes), margin=np.array(margins),
                        block=np.array(blocks), keys=np.stack(keys_all), visible=np.stack(vis_all),
                        pose=np.array(poses), intrinsics=np.array(intrs))


def gen_fusion() -> None:
    """The RC-side fusion behind the sphere fixture (fixtures.py:28-41):
    the 8 frames, intrinsics and config, and per frame the keys
    allocate_blocks created and integrate_frame touched (voxel_model.py:165-299).
    The final TSDF blocks are mc_sphere.npz."""
    from voxelstream.dataset import SphereScene, default_intrinsics, synthetic_frames
    from voxelstream.voxel_model import FusionConfig, VoxelModel

    scene = SphereScene(radius=0.4, orbit_radius=1.4)
    intr = default_intrinsics(80, 60)
    cfg = FusionConfig(voxel_size=0.01, truncation=0.06)
    model = VoxelModel(cfg, bucket_count=1 << 13, excess_capacity=1 << 13)
    depth, color, pose, created, touched = [], [], [], [], []
    for frame in synthetic_frames(scene, intr, 8):
        new = model.allocate_blocks(frame.depth, frame.pose, intr)
        tch = model.integrate_frame(frame.depth, frame.color, frame.pose, intr)
        depth.append(frame.depth)
        color.append(frame.color)
        pose.append(np.concatenate([frame.pose.rotation.reshape(-1), frame.pose.translation]))
        created.append(np.asarray(new, np.int32).reshape(-1, 3))
        touched.append(np.asarray(sorted(tch), np.int32).reshape(-1, 3))
    np.savez_compressed(
        OUT / "fusion_sphere.npz", depth=np.stack(depth).astype(np.float32), color=np.stack(color).astype(np.uint8),
        pose=np.stack(pose).astype(np.float64),
        intr=np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height], np.float64),
        cfg=np.array([cfg.voxel_size, cfg.truncation, cfg.max_weight, cfg.alloc_stride], np.float64),
        created_counts=np.array([len(c) for c in created]), created=np.concatenate(created),
        touched_counts=np.array([len(t) for t in touched]), touched=np.concatenate(touched))


def gen_extract() -> None:
    """BlockHashSet.extract_batch (concurrent_hash.py:366-402): the rotation
    start it draws (random.randrange(capacity) after random.seed(seed)) and
    the keys it returns, over a churned table (excess chains, holes)."""
    out = []
    for seed in range(6):
        s = ch.BlockHashSet(64, 64)
        rng = np.random.default_rng(100 + seed)
        keys = [tuple(int(v) for v in k) for k in rng.integers(-50, 50, (100, 3))]
        for k in keys:
            s.insert(k)
        for k in keys[::3]:
            s.remove(k)
        max_n = [1, 5, 17, 40, 200, 0][seed]
        random.seed(seed)
        start = random.randrange(s.capacity)
        random.seed(seed)
        got = s.extract_batch(max_n)
        out.append({"inserted": [list(k) for k in keys], "removed_every": 3, "max_n": max_n, "start": start,
                    "extracted": [list(k) for k in got], "remaining": sorted(list(k) for k in s.snapshot_keys())})
    (OUT / "extract.json").write_text(json.dumps(out))


def main() -> None:
    gen_hash_kat()
    gen_hash_seq()
    gen_config1()
    gen_mc_random()
    gen_mc_edge()
    gen_mc_sphere()
    gen_stream()
    gen_server()
    gen_visibility()
    gen_fusion()
    gen_extract()
    for p in sorted(OUT.iterdir()):
        if p.suffix in (".json", ".npz"):
            print(f"{p.name:24s} {p.stat().st_size:>9d} B")


if __name__ == "__main__":
    main()
