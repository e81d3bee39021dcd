#!/usr/bin/env python
"""bench.py -- the SLAMCast hot path on B200 (contract: see README/DESIGN.md).

Headline (BASELINE.json configs[1], "config 2"): a 10M-key block hash set at
load factor 0.7, batches of 2^22 mixed ops (50% insert: 40% fresh / 60%
present, 30% find: 50% hit, 20% erase), ONE launch per batch
(vs_table_apply).  A "step" is one batch.  Reported in M ops/s.

Also on the same line (extra objects):
  "mc"     config 3: full MC-index + quantised-TSDF encode of the synthetic
           16 m x 3 m x 16 m room at 5 mm (2,080,160 blocks), blocks/s
  "cpu_baseline"  the C oracle port of the reference algorithm, timed on this
           box's host cores on a bounded sample

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun: every rank owns one hash partition (owner =
fmix32(hash_key) mod N) and each batch is routed to owners with NCCL
all-to-all and back (weak scaling: per-rank batch and live keys fixed).
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "M hash ops/s (insert/find/erase, 1-8 GPU); MC-encoded voxel blocks/s"
BYTES_PER_OP = 43.2   # 0.5*48 + 0.3*32 + 0.2*48 algorithmic bytes per mixed op
BYTES_PER_BLOCK = 8704  # 6144 TSDF read + 2048 MC write + 512 quantised write


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--exchange", default="auto", choices=["auto", "peer", "collective"],
                   help="sharded routing at N>1: kernel peer stores (auto/peer) or NCCL all-to-all")
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--live", type=int, default=None,
                   help="live keys per GPU (default: config 2's 10M at N=1, config 5's 1e9/N at N>1)")
    p.add_argument("--batch-log2", type=int, default=None,
                   help="log2 ops per batch per GPU (default: 22 = config 2 at N=1, 24 = config 5 at N>1)")
    p.add_argument("--config5-slice", type=int, default=0, metavar="G",
                   help="at N=1: run config 5's per-GPU slice for G GPUs (1e9/G live keys, 2^24-op batches)")
    p.add_argument("--no-config1", action="store_true")
    p.add_argument("--bucket-frac", type=float, default=0.5,
                   help="share of the 0.7-load-factor slots in the bucket region (rest: excess)")
    p.add_argument("--mc-steps", type=int, default=10)
    p.add_argument("--no-mc", action="store_true")
    p.add_argument("--no-mc-parity", action="store_true", help="skip the all-blocks oracle check (experiments)")
    p.add_argument("--no-stream", action="store_true")
    p.add_argument("--no-rc", action="store_true")
    p.add_argument("--no-server", action="store_true")
    p.add_argument("--rc-frames", type=int, default=20)
    p.add_argument("--stream-ticks", type=int, default=200)
    p.add_argument("--stream-separate", action="store_true",
                   help="config-4 ticks as three calls (dedup, fan-out, extraction) instead of vs_stream_tick")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-threads", type=int, default=0)
    return p.parse_args()


# --------------------------------------------------------------- helpers

def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str, units: int | None = None):
    """dram bytes per launch of `kernel` from the committed ncu capture --
    only when that capture processed the same number of units per launch
    (ops or blocks) as the launch it is reported beside; else None."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
        for key in (f"{kernel}@{units}", kernel):
            rec = d.get(key)
            if rec and rec.get("units_per_launch") == units:
                return rec.get("dram_bytes_per_launch")
        return None
    except Exception:
        return None


class Clocks:
    """Samples nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "10"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.t:
                self.t.join(timeout=2)
        return self.summary()

    def summary(self):
        import statistics

        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------- CPU (oracle)

def cpu_hash_sample(spec, threads: int, batches: int = 1, seed: int = 0):
    """Oracle port (C restatement of concurrent_hash.py) on a bounded sample:
    build the config-2 table, then time `batches` mixed batches."""
    import numpy as np

    import oracle
    from paper_1805_03709_b200 import workloads

    o = oracle.OracleHashSet(spec.bucket_count, spec.excess)
    chunk = 1 << 22
    for a in range(0, spec.live, chunk):
        o.insert_batch_mt(workloads.id_to_key_np(np.arange(a, min(spec.live, a + chunk))), threads)
    rng = np.random.default_rng(seed)
    lo, hi = 0, spec.live
    times = []
    ok = True
    for step in range(batches):
        ids, ops, expect = workloads.mix_batch_ids_np(spec, step, lo, hi, rng)
        keys = workloads.id_to_key_np(ids)
        t0 = time.perf_counter()
        res, _, fail = o.apply_batch(keys, ops, threads=threads)
        times.append(time.perf_counter() - t0)
        ok &= bool(fail == -1 and np.array_equal(res, expect))
        lo += spec.counts["erase"]
        hi += spec.counts["fresh"]
    return times, ok, o.size()


def cpu_mc_sample(threads: int, n_blocks: int = 32768):
    """Oracle MC encode (C restatement of recompute_mc_block) on a slab of the room."""
    import numpy as np
    import torch

    import oracle
    from paper_1805_03709_b200 import workloads

    keys = workloads.room_block_keys()[:n_blocks]
    rows = workloads.room_tsdf_rows(torch.from_numpy(keys)).numpy()
    nbr = oracle.neighbor_table(keys, keys)
    t0 = time.perf_counter()
    oracle.mc_encode(rows, nbr, threads=threads)
    return time.perf_counter() - t0, n_blocks


# --------------------------------------------------------------- GPU arms

def _free_cuda():
    """Return the previous section's cached blocks (each section sizes its
    own multi-GB pools)."""
    import gc

    import torch

    gc.collect()
    torch.cuda.empty_cache()


def sync_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    import torch

    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()


def run_hash(args, dev, rank, world):
    import torch

    from paper_1805_03709_b200 import BlockHashSet, _lib, workloads

    spec = workloads.MixSpec(live=args.live, load_factor=0.7, batch=1 << args.batch_log2, bucket_frac=args.bucket_frac)
    B = spec.batch
    s = BlockHashSet(spec.bucket_count, spec.excess, device=dev)
    # rank r owns its own id space; with world > 1 keys are routed to owners
    base = rank << 40
    router = None
    if world > 1:
        from paper_1805_03709_b200.shard import ShardedBlockHashSet

        router = ShardedBlockHashSet(s, exchange=args.exchange, max_batch=B)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    # initial fill: `live` keys (routed when sharded)
    chunk = 1 << 22
    for a in range(0, spec.live, chunk):
        ids = torch.arange(base + a, base + min(spec.live, a + chunk), device=dev, dtype=torch.int64)
        keys = workloads.id_to_key_torch(ids)
        if router:
            router.apply(keys, torch.zeros(keys.shape[0], dtype=torch.uint8, device=dev))
        else:
            s.insert_keys(keys)
    s.check_capacity()
    torch.cuda.synchronize()
    lo, hi = base, base + spec.live
    n_total = args.warmup + args.steps
    batches = []
    # e2e window: 3x the timed steps, up to 60 distinct batches and at most
    # ~3 GB of pinned host inputs per rank (config 2: 55 batches, ~60 ms of
    # PCIe-bound transfers; 2^24-op batches: 13), long enough that host-side
    # transients of a few ms do not swing the figure
    n_e2e = 0 if args.no_e2e else max(4, min(3 * args.steps, 60, int(3e9 // (13 * B))))
    for step in range(n_total + n_e2e):
        ids, ops, expect = workloads.mix_batch_ids(spec, step, lo, hi, gen, dev)
        ids = torch.where(ids >= workloads.MISS_BASE, ids + (rank << 50), ids)
        batches.append((workloads.id_to_key_torch(ids), ops, expect))
        lo += spec.counts["erase"]
        hi += spec.counts["fresh"]
    del ids

    def step_fn(i):
        k, o, _ = batches[i]
        if router:
            return router.apply(k, o)
        return s.apply(k, o)[0]

    ok = True
    for i in range(args.warmup):
        r = step_fn(i)
        ok &= bool(torch.equal(r, batches[i][2]))
    s.check_capacity()
    clocks = Clocks(dev.index)
    barrier(world)
    clocks.start()
    time.sleep(0.12)  # let the sampler attach before the region starts
    results = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with _lib.Profile() as prof:
        barrier(world)
        ev0.record()
        for i in range(args.warmup, n_total):
            results.append(step_fn(i))
        ev1.record()
        barrier(world)
    clk = clocks.stop()
    ms = sync_max(ev0.elapsed_time(ev1), world)
    for j, r in enumerate(results):
        ok &= bool(torch.equal(r, batches[args.warmup + j][2]))
    s.check_capacity()
    size_ok = s.approx_size() == spec.live if world == 1 else True
    ops_total = args.steps * B * world
    value = ops_total / (ms / 1e3) / 1e6
    apply_ms = prof.ms["hash"] / max(1, prof.count["hash"])
    # with routing the table sees ~B ops per rank per step as well
    achieved = B * BYTES_PER_OP / (apply_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    # speed of light of the access pattern on this table: dependent random
    # 16-B entry loads only (vs_table_probe_sol), k_apply's launch shape
    import ctypes

    lib = _lib.load()
    probe_out = torch.empty(B, dtype=torch.uint8, device=dev)
    cs = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    sol = {}
    for hops in (1, 2, 3):
        for _ in range(2):
            _lib.check(lib.vs_table_probe_sol(s.handle, B, hops, _lib.ptr(probe_out), cs), "probe")
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        for _ in range(10):
            lib.vs_table_probe_sol(s.handle, B, hops, _lib.ptr(probe_out), cs)
        p1.record()
        torch.cuda.synchronize()
        sol[str(hops)] = hops * B / (p0.elapsed_time(p1) / 10 / 1e3) / 1e9
    del probe_out
    traffic = ncu_traffic("k_apply", B)
    out = {
        "value": value, "ms_per_step": ms / args.steps, "ok": ok and size_ok, "clocks": clk,
        "exchange": router.exchange if router else None,
        "gpu_launches": prof.launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "vsb::k_apply",
                     "kernel_ms": apply_ms, "bytes_per_launch": B * BYTES_PER_OP, "peak_source": peak_src,
                     "traffic_frac": (traffic / (apply_ms / 1e3) / 1e9 / peak) if traffic else None,
                     "random_access_sol": {"g_dependent_entry_loads_per_s": sol,
                                           "probe": "vs_table_probe_sol: 1/2/3 dependent random 16-B entry loads "
                                                    "per op over this table, k_apply's launch shape, no logic"},
                     "note": "algorithmic 43.2 B/op (SURVEY §8d); every 16-B random entry access moves a >= 64-B "
                             "DRAM burst, so the path is bound by DRAM bursts, not bytes: traffic_frac is the "
                             "measured DRAM traffic (ncu, per launch) over the kernel time vs the peak"},
    }
    # ---- e2e through the public API with pinned host buffers: H2D of keys +
    # ops, the apply launch and the D2H of the per-op result flags overlap
    # across steps on three streams (copy-in, compute, copy-out)
    if not args.no_e2e:
        extra = batches[n_total:]
        E = len(extra)
        hk = [b[0].cpu().pin_memory() for b in extra]
        ho = [b[1].cpu().pin_memory() for b in extra]
        hr = [torch.empty(B, dtype=torch.uint8).pin_memory() for _ in extra]
        dk = [torch.empty((B, 3), dtype=torch.int32, device=dev) for _ in range(2)]
        do = [torch.empty(B, dtype=torch.uint8, device=dev) for _ in range(2)]
        comp = torch.cuda.current_stream(dev)
        cin, cout = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        free = [torch.cuda.Event() for _ in range(2)]
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(comp)
        cin.wait_event(e0)
        last = None
        for j in range(E):
            slot = j & 1
            with torch.cuda.stream(cin):
                if j >= 2:
                    cin.wait_event(free[slot])
                dk[slot].copy_(hk[j], non_blocking=True)
                do[slot].copy_(ho[j], non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(cin)
            comp.wait_event(ready)
            res = router.apply(dk[slot], do[slot]) if router else s.apply(dk[slot], do[slot])[0]
            free[slot].record(comp)
            done = torch.cuda.Event()
            done.record(comp)
            with torch.cuda.stream(cout):
                cout.wait_event(done)
                res.record_stream(cout)
                hr[j].copy_(res, non_blocking=True)
                last = torch.cuda.Event()
                last.record(cout)
        comp.wait_event(last)
        e1.record(comp)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e_ms = sync_max(e0.elapsed_time(e1), world)
        e2e_ok = all(torch.equal(hr[j], extra[j][2].cpu()) for j in range(E))
        out["e2e"] = {"value": E * B * world / (e_ms / 1e3) / 1e6, "unit": "M ops/s",
                      "h2d_bytes_per_step": B * 13, "d2h_bytes_per_step": B * 1, "steps": E,
                      "wall_s": wall, "ok": e2e_ok,
                      "note": ("ShardedBlockHashSet.apply" if router else "BlockHashSet.apply") +
                              " on pinned host keys+ops; per-op result flags read back; "
                              "copy-in / compute / copy-out overlapped on three streams"}
    del batches, results
    return out


def run_config1(args, dev):
    """Config 1 (the reference's CPU-runnable case): 100k int3
    keys with ~20% duplicates inserted into BlockHashSet(2^17, 2^17), found
    (with 100k absent probes) and erased, plus the MC encode of 10k random
    blocks.  GPU per step: vs_table_insert + vs_table_find + vs_table_erase
    (400k ops) and one encode launch; beside it the reference algorithm (C
    restatement of concurrent_hash.py:159-295 / mc_encoding.py:118-172) on
    the same inputs on this box's host cores.  Per-op flags are checked
    against the counts the reference gives (80,000 created, 100,000 found +
    100,000 absent, 80,000 erased) on every step, and the MC bytes against
    the oracle once."""
    import numpy as np
    import torch

    import oracle
    from paper_1805_03709_b200 import BlockHashSet, _lib, encode_keys, workloads

    keys, absent = workloads.config1_keys()
    probe = np.concatenate([keys, absent])
    dk = torch.from_numpy(keys).to(dev)
    dp = torch.from_numpy(probe).to(dev)
    s = BlockHashSet(1 << 17, 1 << 17, device=dev)
    n_ops = len(keys) * 2 + len(probe)
    expect_found = torch.cat([torch.ones(len(keys), dtype=torch.uint8), torch.zeros(len(absent), dtype=torch.uint8)])

    def step(k, p):
        c, _ = s.insert_keys(k)
        f, _ = s.find_keys(p)
        e, _ = s.erase_keys(k)
        return c, f, e

    def check(c, f, e):
        return (int(c.sum()) == 80_000 and torch.equal(f.cpu(), expect_found) and int(e.sum()) == 80_000)

    ok = True
    for _ in range(3):
        ok &= check(*step(dk, dp))
    for _ in range(20):  # settle clocks / allocator (the steps are ~0.15 ms each)
        step(dk, dp)
    steps = 200
    # keep only the last steps' outputs: holding all 200 steps' result
    # tensors (~2 MB each) made the caching allocator cudaMalloc new segments
    # inside the timed loop (synchronous, ms each: 0.6-4.8 ms steps)
    from collections import deque

    res = deque(maxlen=3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with _lib.Profile(events=False) as prof:
        e0.record()
        for _ in range(steps):
            res.append(step(dk, dp))
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ok &= all(check(*r) for r in res)
    ok &= s.approx_size() == 0
    # e2e: pinned host keys in, the three flag vectors out, every step
    hk, hp = torch.from_numpy(keys).pin_memory(), torch.from_numpy(probe).pin_memory()
    hc = torch.empty(len(keys), dtype=torch.uint8).pin_memory()
    hf = torch.empty(len(probe), dtype=torch.uint8).pin_memory()
    he = torch.empty(len(keys), dtype=torch.uint8).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    for _ in range(steps):
        c, f, e = step(hk.to(dev, non_blocking=True), hp.to(dev, non_blocking=True))
        hc.copy_(c, non_blocking=True)
        hf.copy_(f, non_blocking=True)
        he.copy_(e, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / steps
    ok &= check(hc, hf, he)
    # MC: 10k blocks, field (a) of SURVEY §8d, one encode launch per step
    mkeys = workloads.config1_mc_keys()
    tsdf, weight, color = workloads.random_field(len(mkeys))
    rows = oracle.make_pool(tsdf, weight, color)
    t = BlockHashSet(1 << 14, 1 << 14, device=dev)
    dmk = torch.from_numpy(mkeys).to(dev)
    _, pos = t.insert_keys(dmk)
    pool = torch.zeros((t.capacity, 6144), dtype=torch.uint8, device=dev)
    pool[pos.long()] = torch.from_numpy(rows).to(dev)
    mc = torch.empty((len(mkeys), 2048), dtype=torch.uint8, device=dev)
    q = torch.empty((len(mkeys), 512), dtype=torch.int8, device=dev)
    cnt = torch.empty(len(mkeys), dtype=torch.int32, device=dev)
    for _ in range(3):
        encode_keys(t, pool, dmk, mc=mc, q=q, counts=cnt)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        encode_keys(t, pool, dmk, mc=mc, q=q, counts=cnt)
    e1.record()
    torch.cuda.synchronize()
    mc_ms = e0.elapsed_time(e1) / steps
    nbr = oracle.neighbor_table(mkeys, mkeys)
    omc, oq, _ = oracle.mc_encode(rows, nbr, threads=1)
    mc_ok = bool(np.array_equal(mc.cpu().numpy(), omc) and np.array_equal(q.cpu().numpy(), oq))
    # the reference algorithm on the host, same inputs: the C restatement
    # (sequential, one thread, like the reference under the GIL)
    o = oracle.OracleHashSet(1 << 17, 1 << 17)
    ct = []
    for _ in range(3):
        a = time.perf_counter()
        oc = o.insert_batch(keys)[0]
        of = o.find_batch(probe)[0]
        oe = o.erase_batch(keys)[0]
        ct.append(time.perf_counter() - a)
    cpu_ok = bool(int(oc.sum()) == 80_000 and int(of.sum()) == 100_000 and int(oe.sum()) == 80_000)
    a = time.perf_counter()
    oracle.mc_encode(rows, nbr, threads=1)
    cpu_mc_s = time.perf_counter() - a
    return {"workload": "config 1: 100k int3 keys (~20% duplicates) insert + find (with 100k absent probes) + "
                        "erase on BlockHashSet(2^17, 2^17); MC + quantised encode of 10k random 8^3 blocks",
            "hash": {"value": n_ops / (ms / 1e3) / 1e6, "unit": "M ops/s", "ms_per_step": ms, "ops_per_step": n_ops,
                     "gpu_launches_per_step": prof.launches / steps,
                     "e2e": {"value": n_ops / (e2e_ms / 1e3) / 1e6, "unit": "M ops/s",
                             "h2d_bytes_per_step": (len(keys) + len(probe)) * 12,
                             "d2h_bytes_per_step": len(keys) * 2 + len(probe),
                             "note": "pinned host keys -> device, the three BlockHashSet calls, flags -> host"}},
            "mc": {"value": len(mkeys) / (mc_ms / 1e3), "unit": "blocks/s", "ms_per_step": mc_ms, "ok": mc_ok},
            "ok": bool(ok),
            "cpu_reference": {"hash": {"value": n_ops / min(ct) / 1e6, "unit": "M ops/s", "cores": 1, "kind": "port",
                                       "ok": cpu_ok},
                              "mc": {"value": len(mkeys) / cpu_mc_s, "unit": "blocks/s", "cores": 1, "kind": "port"},
                              "sample": "the whole config-1 workload (C restatement of the reference algorithm, "
                                        "sequential, one thread); the reference Python itself measured 0.40/0.82/0.38 "
                                        "M ops/s and 8.6k blocks/s/core (SURVEY §6)"}}


def mc_full_parity(t, pool, keys, mc, q, counts, threads: int, chunk: int = 1 << 17):
    """Every block of the config-3 encode vs the C oracle (recompute_mc_block
    restated), outside the timed region: per chunk, the neighbour rows are
    gathered from the device pool and re-encoded on the host cores."""
    import numpy as np
    import torch

    import oracle
    from paper_1805_03709_b200 import neighbors

    N = keys.shape[0]
    bad = 0
    for a in range(0, N, chunk):
        b = min(N, a + chunk)
        nbr = neighbors(t, keys[a:b]).reshape(-1)
        valid = nbr >= 0
        uniq, inv = torch.unique(nbr[valid], return_inverse=True)
        rows = pool[uniq.long()].cpu().numpy()
        local = torch.full_like(nbr, -1)
        local[valid] = inv.to(torch.int32)
        omc, oq, oc = oracle.mc_encode(rows, local.view(-1, 8).cpu().numpy(), threads=threads)
        ok = (np.array_equal(mc[a:b].cpu().numpy(), omc) and np.array_equal(q[a:b].cpu().numpy(), oq)
              and np.array_equal(counts[a:b].cpu().numpy().astype(np.uint32), oc))
        bad += 0 if ok else 1
    return bad == 0


def run_mc(args, dev, world=1):
    """Config 3: full encode of the synthetic room (2,080,160 blocks).  With
    world > 1 every rank encodes its own replica of the scene (the encoder
    does not shard): value = world x blocks / max-over-ranks time.

    Headline: ONE self-contained launch per step (vs_mc_encode_keys: fused
    neighbour lookups, centre rows by TMA, the 217 halo voxels gathered one
    block ahead, MC + quantised TSDF + counts).  Also timed: the same launch
    with the fused cell compaction, the incremental-ingest variant (face-pack
    side table rebuilt for every row by k_mc_faces, then the encode reading
    it: both kernels inside the timed region), and the two-pass compaction."""
    import numpy as np
    import torch

    from paper_1805_03709_b200 import BlockHashSet, _lib, compact, encode_keys, face_packs, workloads

    keys_np = workloads.room_block_keys()
    N = len(keys_np)
    keys = torch.from_numpy(keys_np).to(dev)
    # the normative spatial hash (concurrent_hash.py:49-59) collides heavily on
    # structured room keys (1.35M distinct values for 2.08M keys): ~1.08M keys
    # land in the excess region whatever the bucket count, so size it 2^21
    t = BlockHashSet(1 << 21, 1 << 21, device=dev)
    _, pos = t.insert_keys(keys)
    t.check_capacity()
    pool = torch.empty((t.capacity, 6144), dtype=torch.uint8, device=dev)
    for a in range(0, N, 1 << 15):
        pool[pos[a:a + (1 << 15)].long()] = workloads.room_tsdf_rows(keys[a:a + (1 << 15)])
    mc = torch.empty((N, 2048), dtype=torch.uint8, device=dev)
    q = torch.empty((N, 512), dtype=torch.int8, device=dev)
    cnt = torch.empty(N, dtype=torch.int32, device=dev)

    def enc():
        return encode_keys(t, pool, keys, mc=mc, q=q, counts=cnt)

    for _ in range(2):
        enc()
    torch.cuda.synchronize()

    def timed(fn, steps):
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with _lib.Profile() as prof:
            e0.record()
            for _ in range(steps):
                fn()
            e1.record()
            barrier(world)
        return sync_max(e0.elapsed_time(e1), world) / steps, prof

    clocks = Clocks(dev.index).start()
    time.sleep(0.12)
    ms, prof = timed(enc, args.mc_steps)
    clk = clocks.stop()
    k_ms = prof.ms["mc"] / max(1, prof.count["mc"])
    launches = prof.launches
    # ---- parity of EVERY block vs the C oracle (outside the timed region)
    mc_t, q_t, c_t = enc()
    torch.cuda.synchronize()
    p0 = time.perf_counter()
    ok = None if args.no_mc_parity else mc_full_parity(t, pool, keys, mc_t, q_t, c_t, threads=cpu_cores())
    parity_s = time.perf_counter() - p0
    # ---- the same launch with the fused compaction of the non-empty cells
    total_cells = int(c_t.long().sum().item())
    cap = total_cells + 1024
    cstate = {}

    def enc_cells():
        cstate["r"] = encode_keys(t, pool, keys, mc=mc, q=q, counts=cnt, cells=True, cell_cap=cap)

    enc_cells()
    c_ms, c_prof = timed(enc_cells, args.mc_steps)
    _, _, c_counts, (offs, flat, cells, cur) = cstate["r"]
    cells_ok = bool(int(cur.item()) == total_cells and torch.equal(c_counts, c_t))
    if cells_ok:  # scatter-back of every block's cells == dense MC bytes
        cl = c_counts.long()
        blk = torch.repeat_interleave(torch.arange(N, device=dev), cl)
        src = torch.repeat_interleave(offs.long(), cl) + torch.arange(total_cells, device=dev) - \
            torch.repeat_interleave(torch.cumsum(cl, 0) - cl, cl)
        dense = torch.zeros((N, 512), dtype=torch.int32, device=dev)
        dense[blk, flat[src].long() & 0xFFFF] = cells[src]
        cells_ok = bool(torch.equal(dense.view(torch.uint8).view(N, 2048), mc_t))
        del dense, blk, src
    # ---- incremental-ingest variant: side-table rebuild of every row + encode
    faces = face_packs(pool, rows=pos)

    def enc_packs():
        face_packs(pool, rows=pos, faces=faces)
        encode_keys(t, pool, keys, mc=mc, q=q, counts=cnt, faces=faces)

    p_ms, _ = timed(enc_packs, max(2, args.mc_steps // 2))
    f_ms, f_prof = timed(lambda: encode_keys(t, pool, keys, mc=mc, q=q, counts=cnt, faces=faces),
                         max(2, args.mc_steps // 2))

    def two_pass():
        m, _, c = encode_keys(t, pool, keys, mc=mc, q=False, counts=cnt)
        compact(m, c, cell_cap=cap)

    tp_ms, _ = timed(two_pass, 2)
    peak, src = peaks()
    achieved = N * BYTES_PER_BLOCK / (k_ms / 1e3) / 1e9
    cell_bytes = total_cells * 6
    ck_ms = c_prof.ms["mc"] / max(1, c_prof.count["mc"])
    out = {"workload": "config 3: room 16x3x16 m, 5 mm voxels, 2,080,160 blocks; full encode in ONE self-contained "
                       "launch (fused hash lookups, TMA centre rows, halo voxels gathered one block ahead, MC + "
                       "quantised TSDF + counts)" + (f"; one replica per GPU x{world}" if world > 1 else ""),
           "value": world * N / (ms / 1e3), "unit": "blocks/s", "ms_per_step": ms,
           "steps": args.mc_steps, "blocks": N, "ok": ok,
           "parity": None if ok is None else f"all {N} blocks (MC bytes, quantised bytes, counts) vs the C oracle "
                                             f"on {cpu_cores()} host threads, {parity_s:.1f} s",
           "gpu_launches": launches, "clocks": clk,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "traffic": ncu_traffic("k_mc_encode", N), "kernel": "vsb::k_mc_encode<true,false,false>",
                        "kernel_ms": k_ms, "bytes_per_launch": N * BYTES_PER_BLOCK, "peak_source": src,
                        "bytes_per_block": "6144 TSDF read + 2048 MC + 512 quantised (SURVEY §8d)"},
           "compact": {"value": world * N / (c_ms / 1e3), "unit": "blocks/s", "ms_per_step": c_ms,
                       "cells": total_cells, "ok": cells_ok, "kernel_ms": ck_ms,
                       "frac": (N * BYTES_PER_BLOCK + cell_bytes) / (ck_ms / 1e3) / 1e9 / peak,
                       "note": "the same launch + fused compaction of the non-empty cells (u16 flat + u32 cell; one "
                               "atomic range reservation per block); frac counts +6 B per cell; checked by "
                               "scatter-back of every block"},
           "incremental_packs": {"ms_per_step": p_ms, "value": world * N / (p_ms / 1e3),
                                 "encode_only_ms": f_ms,
                                 "note": "ingest-maintained variant (GpuServerCore): k_mc_faces rebuilds the face "
                                         "bit-packs of ALL rows + the encode reading them, both timed; "
                                         "encode_only_ms = the encode alone when packs are current"},
           "two_pass_compact_ms": tp_ms}
    if not args.no_e2e:
        # e2e: host TSDF rows -> device pool, encode, MC + quantised bytes ->
        # host, pipelined in chunks of the key order on three streams: the
        # upload of chunk c+1 and the download of chunk c-1 overlap the encode
        # of chunk c, which starts once chunk c+1 is resident (its +x/+y/+z
        # halo lies at most ~5k blocks ahead in key order)
        # one rank alone: the whole scene; N > 1 ranks share the host, so each
        # streams its first 2^18 blocks (the full scene would pin ~18 GB per rank)
        Ne = N if world == 1 else min(N, 1 << 18)
        host_rows = pool[pos[:Ne].long()].cpu().pin_memory()
        h_mc = torch.empty((Ne, 2048), dtype=torch.uint8).pin_memory()
        h_q = torch.empty((Ne, 512), dtype=torch.int8).pin_memory()
        posl = pos[:Ne].long()
        nch = 16
        bounds = [Ne * c // nch for c in range(nch + 1)]
        cmax = max(bounds[c + 1] - bounds[c] for c in range(nch))
        stage = [torch.empty((cmax, 6144), dtype=torch.uint8, device=dev) for _ in range(2)]
        comp = torch.cuda.current_stream(dev)
        cin, cout = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 2
        e0.record(comp)
        cin.wait_stream(comp)
        for _ in range(steps):
            ready = []
            for c in range(nch + 1):
                if c < nch:
                    a, b = bounds[c], bounds[c + 1]
                    with torch.cuda.stream(cin):
                        st_ = stage[c & 1][: b - a]
                        st_.copy_(host_rows[a:b], non_blocking=True)
                        pool.index_copy_(0, posl[a:b], st_)
                        ev = torch.cuda.Event()
                        ev.record(cin)
                        ready.append(ev)
                if c >= 1:
                    a, b = bounds[c - 1], bounds[c]
                    comp.wait_event(ready[c] if c < nch else ready[c - 1])
                    encode_keys(t, pool, keys[a:b], mc=mc[a:b], q=q[a:b], counts=False)
                    done = torch.cuda.Event()
                    done.record(comp)
                    with torch.cuda.stream(cout):
                        cout.wait_event(done)
                        h_mc[a:b].copy_(mc[a:b], non_blocking=True)
                        h_q[a:b].copy_(q[a:b], non_blocking=True)
            # the next step's uploads overwrite pool rows the encode still reads
            cin.wait_stream(comp)
        comp.wait_stream(cout)
        e1.record(comp)
        barrier(world)
        e_ms = sync_max(e0.elapsed_time(e1), world)
        torch.cuda.synchronize()
        e2e_ok = bool(torch.equal(h_mc[:4096], mc[:4096].cpu()) and torch.equal(h_q[-4096:], q[Ne - 4096:Ne].cpu()))
        del stage
        out["e2e"] = {"value": world * Ne * steps / (e_ms / 1e3), "unit": "blocks/s", "h2d_bytes_per_step": Ne * 6144,
                      "d2h_bytes_per_step": Ne * (2048 + 512), "steps": steps, "ok": e2e_ok, "blocks_per_rank": Ne,
                      "note": "pinned host rows -> pool, encode, MC + quantised bytes -> pinned host; 16 chunks "
                              "pipelined on three streams (upload / encode / download)"}
    return out


STREAM_C, STREAM_U, STREAM_X, STREAM_K, STREAM_EVERY = 16, 512, 512, 256, 20
BYTES_PER_STREAM_INSERT = 48  # one hash insert per (client, key)


def stream_script(keys_np, ticks: int, seed: int = 44):
    """Config-4 tick script (host copy, identical for the GPU run, the
    oracle replay and the CPU baseline): updated keys per tick and reset
    keys per reconnect tick."""
    import numpy as np

    rng = np.random.default_rng(seed)
    M = len(keys_np)
    upd = keys_np[rng.integers(0, M, (ticks + 1) * STREAM_U)].reshape(ticks + 1, STREAM_U, 3)
    resets = keys_np[rng.integers(0, M, (ticks // STREAM_EVERY + 1) * STREAM_K)].reshape(-1, STREAM_K, 3)
    return np.ascontiguousarray(upd), np.ascontiguousarray(resets)


def stream_replay_client(c, scene, aff, resets, ticks, extracted=None, seed=0):
    """One client of the config-4 script on the CPU: the reference StreamSet
    semantics (server.py:49-95) over the C restatement of BlockHashSet --
    created = the set difference, appended to the generation FIFO in order;
    extract_batch either ADOPTS the keys the GPU extracted (parity: they must
    be pending and as many as min(512, size)) or runs the port's own
    extraction (CPU baseline).  Returns (table, fifo parts, key-ops, ok)."""
    import numpy as np

    import oracle

    o = oracle.OracleHashSet(1 << 21, 1 << 21)
    cr, _, _ = o.insert_batch(scene)
    fifo = [scene[cr.astype(bool)]]
    ops, ok = len(scene), True
    rs = np.random.default_rng(seed)
    for t in range(ticks + 1):
        a = aff[t]
        cr, _, fail = o.insert_batch(a)
        ok &= fail == -1
        fifo.append(a[cr.astype(bool)])
        ops += len(a)
        if extracted is not None:
            ex = extracted[t]
            want = min(STREAM_X, o.size())
            er, _ = o.erase_batch(ex)
            ok &= bool(er.all()) and len(ex) == want
        else:
            ex = o.extract(STREAM_X, int(rs.integers(0, o.capacity)))
        ops += len(ex)
        if t % STREAM_EVERY == STREAM_EVERY - 1:
            if (t // STREAM_EVERY) % STREAM_C == c:  # fresh reconnect: clear + fill
                o.clear()
                cr, _, _ = o.insert_batch(scene)
                fifo = [scene[cr.astype(bool)]]
                ops += len(scene)
            o.erase_batch(resets[t // STREAM_EVERY])
            ops += STREAM_K
    return o, fifo, ops, ok


def run_stream(args, dev):
    """Config 4: 16 clients' stream sets over the 2.08M-block room scene.

    Fresh fill of every client, then `ticks` ticks of: 512 random updated
    TSDF keys -> affected dedup -> insert into all 16 sets (one launch) ->
    every client extract_random(512).  Every 20 ticks one client reconnects
    fresh (clear + full fill) and a reset of 256 keys is removed from every
    set.  Unit: stream-set key ops (inserts + removals) per second.  After
    the timed script every client's sorted pending set and FIFO are compared
    with a replay of the same script on the CPU restatement."""
    import ctypes
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np
    import torch

    import oracle
    from paper_1805_03709_b200 import (BlockHashSet, StreamSet, _lib, extract_random_many, fan_out,
                                       remove_everywhere, stream_tick, workloads)

    scene_np = workloads.room_block_keys()
    keys = torch.from_numpy(scene_np).to(dev)
    M = keys.shape[0]
    C, U, X, K = STREAM_C, STREAM_U, STREAM_X, STREAM_K
    ticks = max(args.stream_ticks, STREAM_EVERY)
    upd_np, resets_np = stream_script(scene_np, ticks)
    clients = [StreamSet(1 << 21, 1 << 21, device=dev, fifo_capacity=1 << 22) for _ in range(C)]
    scratch = BlockHashSet(1 << 14, 1 << 14, device=dev)
    lib = _lib.load()
    # device-side logs (read once after the timed region): affected keys and
    # counts per tick, extracted keys and counts per tick and client
    aff_keys = torch.zeros((ticks + 1, 8 * U, 3), dtype=torch.int32, device=dev)
    aff_log = torch.zeros((ticks + 1, 1), dtype=torch.int64, device=dev)
    ex_keys = torch.zeros((ticks + 1, C, X, 3), dtype=torch.int32, device=dev)
    ex_log = torch.zeros((ticks + 1, C), dtype=torch.int64, device=dev)
    # inputs resident in HBM before the timed region, as in the other sections
    upd_all = torch.from_numpy(upd_np).to(dev)
    reset_all = torch.from_numpy(resets_np).to(dev)
    seeds = [[(t * C + c) * 2654435761 + 17 for c in range(C)] for t in range(ticks + 1)]

    def tick(t):
        if not args.stream_separate:
            # ONE launch: dedup -> fan-out into all 16 sets -> 16 extractions
            stream_tick(clients, upd_all[t], X, seeds[t], affected_out=aff_keys[t], n_affected=aff_log[t],
                        keys_out=ex_keys[t], n_out=ex_log[t])
        else:
            st = torch.cuda.current_stream(dev)
            _lib.check(lib.vs_affected_dedup(scratch.handle, _lib.ptr(upd_all[t]), U, _lib.ptr(aff_keys[t]),
                                             _lib.ptr(aff_log[t]), ctypes.c_void_p(st.cuda_stream)))
            # no host sync: the fan-out (one launch, k_multi_fan_small) takes the
            # device-side affected count
            fan_out(clients, aff_keys[t], sync=False, n_dev=aff_log[t])
            extract_random_many(clients, X, seeds[t], n_out=ex_log[t], keys_out=ex_keys[t])  # one launch
        if t % STREAM_EVERY == STREAM_EVERY - 1:
            victim = clients[(t // STREAM_EVERY) % C]
            victim.clear()
            fan_out([victim], keys, sync=False)
            remove_everywhere(clients, reset_all[t // STREAM_EVERY])

    # one untimed fill + clear first: the FIFO rings and the fan-out's ~400 MB
    # of stream-ordered scratch are then already mapped (one-time growth of
    # the allocator's pool, not part of a fill); the clients are empty again
    fan_out(clients, keys)
    for c in clients:
        c.clear()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    fan_out(clients, keys)  # fresh fill of all 16 clients: 16 x 2.08M inserts, one launch
    f1.record()
    torch.cuda.synchronize()
    fill_ms = f0.elapsed_time(f1)
    ok = all(c.size() == M for c in clients)
    tick(0)
    torch.cuda.synchronize()
    clocks = Clocks(dev.index).start()
    time.sleep(0.12)
    t0 = time.perf_counter()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(ticks + 1)]
    with _lib.Profile(events=False) as prof:
        for t in range(1, ticks + 1):
            evs[t - 1].record()
            tick(t)
        evs[ticks].record()
        torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    clk = clocks.stop()
    ms = evs[0].elapsed_time(evs[ticks])
    per_tick = [evs[t - 1].elapsed_time(evs[t]) for t in range(1, ticks + 1)]
    aff_n = aff_log[:, 0].cpu().numpy()
    ex_n = ex_log.cpu().numpy()
    reconnect = {t for t in range(1, ticks + 1) if t % STREAM_EVERY == STREAM_EVERY - 1}
    ins = int(C * aff_n[1:].sum()) + len(reconnect) * M
    rem = int(ex_n[1:].sum()) + len(reconnect) * C * K
    total = ins + rem
    plain = [t for t in range(1, ticks + 1) if t not in reconnect]
    plain_ms = sum(per_tick[t - 1] for t in plain)
    plain_ops = int(sum(C * aff_n[t] + ex_n[t].sum() for t in plain))
    # ---- parity: replay the same script on the CPU restatement, adopting
    # the GPU's extracted keys; compare every client's sorted pending set and
    # its FIFO (stale entries included) -- outside the timed region
    p0 = time.perf_counter()
    aff_host = [aff_keys[t, : int(aff_n[t])].cpu().numpy() for t in range(ticks + 1)]
    ex_host = ex_keys.cpu().numpy()
    dedup_ok = True
    for t in (0, 1, ticks // 2, ticks):  # the GPU affected dedup vs the reference's dict order
        want = np.array(oracle.affected_dedup(upd_np[t].tolist()), np.int32).reshape(-1, 3)
        dedup_ok &= bool(np.array_equal(aff_host[t], want))

    def check_client(c):
        o, fifo, _, rok = stream_replay_client(
            c, scene_np, aff_host, resets_np, ticks,
            extracted=[ex_host[t, c, : int(ex_n[t, c])] for t in range(ticks + 1)])
        want_keys = o.snapshot()[0]
        want_keys = want_keys[np.lexsort(want_keys.T[::-1])]
        return rok, want_keys, np.concatenate(fifo)

    with ThreadPoolExecutor(max_workers=min(C, cpu_cores())) as ex:
        replays = list(ex.map(check_client, range(C)))
    parity_ok = dedup_ok
    bad = []
    for c, (rok, want_keys, want_fifo) in enumerate(replays):
        got = clients[c]._set.snapshot_tensor()[0].cpu().numpy()
        got = got[np.lexsort(got.T[::-1])]
        fifo = clients[c]._ring_view().cpu().numpy()
        good = (bool(rok), bool(np.array_equal(got, want_keys)), bool(np.array_equal(fifo, want_fifo)))
        parity_ok &= all(good)
        if not all(good):
            bad.append({"client": c, "replay_ok/set/fifo": good, "sizes": [len(got), len(want_keys)],
                        "fifo_len": [len(fifo), len(want_fifo)]})
    parity_s = time.perf_counter() - p0
    # ---- roofline of the fan-out (the dominant launch chain of a tick):
    # 48 B per (client, key) insert, timed alone on a tick's affected keys
    A = int(aff_n[1])
    for _ in range(3):
        fan_out(clients, aff_keys[1, :A], sync=False)
    torch.cuda.synchronize()
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    r0.record()
    for _ in range(reps):
        fan_out(clients, aff_keys[1, :A], sync=False)
    r1.record()
    torch.cuda.synchronize()
    fan_ms = r0.elapsed_time(r1) / reps
    peak, src = peaks()
    fan_bytes = C * A * BYTES_PER_STREAM_INSERT
    return {"workload": "config 4: 16 clients x 2,080,160-block scene; per tick 512 updated TSDF keys -> "
                        "affected dedup -> insert into all sets, extract_random(512) per client; every 20 ticks a "
                        "fresh reconnect (clear + full fill) and a 256-key reset from every set",
            "value": total / (ms / 1e3) / 1e6, "unit": "M key-ops/s", "ticks": ticks,
            "ms_per_tick": ms / ticks, "wall_s": wall, "fill_16_clients_ms": fill_ms,
            "fill_value": C * M / (fill_ms / 1e3) / 1e6, "inserts": ins, "removes": rem,
            "tick_only": {"value": plain_ops / (plain_ms / 1e3) / 1e6, "unit": "M key-ops/s",
                          "ms_per_tick": plain_ms / len(plain), "ticks": len(plain),
                          "note": "ticks without a reconnect fill / reset: dedup + 16-client fan-out + 16 extracts"},
            "ok": bool(ok and parity_ok), "parity_bad_clients": bad[:3],
            "parity": f"all {C} clients: sorted pending set + FIFO (stale entries included) after the script == a "
                      f"replay on the C restatement adopting the GPU's extracted keys; affected dedup == the "
                      f"reference's dict order ({parity_s:.1f} s)",
            "gpu_launches": prof.launches, "clocks": clk,
            "roofline": {"bound": "hbm", "kernel": "fan-out (k_multi_fan_small: inserts + fixup + scan + FIFO append)",
                         "achieved": fan_bytes / (fan_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": fan_bytes / (fan_ms / 1e3) / 1e9 / peak, "traffic": None, "kernel_ms": fan_ms,
                         "bytes_per_launch": fan_bytes, "peak_source": src,
                         "note": f"48 B per (client, key) insert (SURVEY §8d) x {C} clients x {A} affected keys; "
                                 "latency-bound: a tick's fan-out is ~65k inserts"},
            "tick_path": ("3 launches per tick: k_dedup_small -> k_multi_fan_small -> k_multi_extract"
                          if args.stream_separate else
                          "ONE launch per tick (vs_stream_tick): per client one CTA runs the affected dedup, "
                          "the fan-out (inserts, created fixup, block scan, FIFO append) and its extraction"),
            "note": "inserts count created-or-not key inserts into every set; removes = extracted + reset keys; "
                    "no host sync inside a tick (device-side affected count bounds the fan-out)"}


def cpu_stream_baseline(threads: int, ticks: int):
    """The same 16-client tick script on the CPU port (C restatement of
    BlockHashSet + the StreamSet FIFO rule, own extraction), one host thread
    per client (clients are independent), wall-clock timed."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle
    from paper_1805_03709_b200 import workloads

    scene = workloads.room_block_keys()
    upd, resets = stream_script(scene, ticks)
    t0 = time.perf_counter()
    aff = [np.array(oracle.affected_dedup(upd[t].tolist()), np.int32).reshape(-1, 3) for t in range(ticks + 1)]
    with ThreadPoolExecutor(max_workers=min(STREAM_C, threads)) as ex:
        res = list(ex.map(lambda c: stream_replay_client(c, scene, aff, resets, ticks, seed=c)[2], range(STREAM_C)))
    dt = time.perf_counter() - t0
    return sum(res) / dt / 1e6, dt


def run_server(args, dev):
    """SURVEY §3.1, the core server path end to end through
    GpuServerCore.on_tsdf_batch (server.py:299-315): per tick 512 updated
    TSDF blocks (wire rows, resident in HBM) -> tsdf_map.put (latest write
    wins) + face packs of the written rows -> affected dedup (~4k MC keys)
    -> mc_map.put + recompute straight into the MC / quantised pools ->
    fan-out into 16 exploration clients.  The scene (2,080,160 blocks) is
    ingested first and 16 clients attach fresh."""
    import numpy as np
    import torch

    import oracle
    from paper_1805_03709_b200 import GpuServerCore, _lib, neighbors, workloads

    scene_np = workloads.room_block_keys()
    scene = torch.from_numpy(scene_np).to(dev)
    M = scene.shape[0]
    core = GpuServerCore(1 << 21, 1 << 21, stream_buckets=1 << 21, stream_excess=1 << 21, max_batch=1 << 16,
                         device=dev)
    torch.cuda.synchronize()
    i0 = time.perf_counter()
    chunk = 1 << 16
    for a in range(0, M, chunk):
        k = scene[a:a + chunk]
        core.on_tsdf_batch(k, workloads.room_tsdf_rows(k), sync=False)
    core.check()
    torch.cuda.synchronize()
    ingest_s = time.perf_counter() - i0
    C = STREAM_C
    for c in range(C):
        core.attach(bytes([c]) * 16)
    torch.cuda.synchronize()
    T = max(20, args.stream_ticks // 2)
    Ts = 5
    rng = np.random.default_rng(77)
    upd_np = scene_np[rng.integers(0, M, (T + Ts + 3) * STREAM_U)].reshape(T + Ts + 3, STREAM_U, 3)
    upd = torch.from_numpy(upd_np).to(dev)
    # updated rows: the scene's rows with every tsdf value nudged (a real update)
    rows = []
    for t in range(T + Ts + 3):
        r = workloads.room_tsdf_rows(upd[t]).view(torch.float32).view(STREAM_U, 512, 3)
        r[..., 0] = (r[..., 0] * 0.97).clamp(-1, 1)
        rows.append(r.reshape(STREAM_U, -1).view(torch.uint8).reshape(STREAM_U, 6144))
    rows = torch.stack(rows)
    for t in range(3):  # warm-up
        core.on_tsdf_batch(upd[t], rows[t], sync=False)
    torch.cuda.synchronize()
    clocks = Clocks(dev.index).start()
    time.sleep(0.12)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    with _lib.Profile(events=False) as prof:
        e0.record()
        for t in range(3, 3 + T):
            core.on_tsdf_batch(upd[t], rows[t], sync=False)
        e1.record()
        host_s = time.perf_counter() - h0
        torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / T
    core.check()
    # the exact path (reference failure semantics, three host syncs per tick)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for t in range(3 + T, 3 + T + Ts):
        core.on_tsdf_batch(upd[t], rows[t], sync=True)
    s1.record()
    torch.cuda.synchronize()
    ms_sync = s0.elapsed_time(s1) / Ts
    # parity: the MC + quantised bytes of the last tick's affected keys in the
    # pools == the oracle re-encode of the same keys from the device TSDF
    # pool; the affected set == the reference's dict-order dedup
    aff = np.array(oracle.affected_dedup(upd_np[3 + T + Ts - 1].tolist()), np.int32).reshape(-1, 3)
    found, mpos = core.mc_map.find_keys(aff)
    nbr = neighbors(core.tsdf_map, aff).reshape(-1)
    valid = nbr >= 0
    uniq, inv = torch.unique(nbr[valid], return_inverse=True)
    trows = core.tsdf_pool[uniq.long()].cpu().numpy()
    local = torch.full_like(nbr, -1)
    local[valid] = inv.to(torch.int32)
    omc, oq, _ = oracle.mc_encode(trows, local.view(-1, 8).cpu().numpy(), threads=8)
    ok = bool(found.all().item()) and np.array_equal(core.mc_pool[mpos.long()].cpu().numpy(), omc) and \
        np.array_equal(core.q_pool[mpos.long()].cpu().numpy(), oq)
    ok &= all(st.size() <= core.mc_map.approx_size() for st in core.streams())
    return {"workload": f"SURVEY §3.1 on_tsdf_batch: {STREAM_U} updated TSDF blocks per tick over the 2,080,160-block "
                        f"room, ~{len(aff)} affected MC keys re-encoded into the MC pool, fan-out to {C} clients",
            "value": 1e3 / ms, "unit": "ticks/s", "ms_per_tick": ms, "ticks": T,
            "blocks_per_s": STREAM_U / (ms / 1e3), "host_ms_per_tick": 1e3 * host_s / T,
            "ms_per_tick_exact_path": ms_sync,
            "note_exact_path": "sync=True: the reference's sequential CapacityExhausted semantics (3 host syncs)",
            "ingest_scene_s": ingest_s, "ok": ok, "gpu_launches": prof.launches, "clocks": clk,
            "parity": "last tick's affected keys: MC + quantised pool bytes == oracle re-encode; affected set == "
                      "the reference's dict-order dedup"}


def run_rc(args, dev):
    """RC-side voxel hashing: allocate_blocks +
    integrate_frame of 640x480 RGB-D frames from inside the synthetic room at
    5 mm voxels (mu 0.06 m), frames resident on the device."""
    import torch

    from paper_1805_03709_b200 import _lib, workloads
    from paper_1805_03709_b200.voxel_model import GpuVoxelModel

    import types

    n = args.rc_frames
    depth, color, Rs, ts, (fx, fy, cx, cy, w, h) = workloads.room_frames(n + 2, 640, 480)
    intr = types.SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)
    cfg = types.SimpleNamespace(voxel_size=0.005, truncation=0.06, max_weight=128.0, alloc_stride=1)
    model = GpuVoxelModel(cfg, bucket_count=1 << 21, excess_capacity=1 << 21, device=dev)
    dd = torch.from_numpy(depth).to(dev)
    cc = torch.from_numpy(color).to(dev)
    for f in range(2):  # warm-up frames
        model.allocate_blocks_tensor(dd[f], (Rs[f], ts[f]), intr)
        model.integrate_frame_tensor(dd[f], cc[f], (Rs[f], ts[f]), intr)
    torch.cuda.synchronize()
    created = touched = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    with _lib.Profile() as prof:
        e0.record()
        for f in range(2, n + 2):
            created += model.allocate_blocks_tensor(dd[f], (Rs[f], ts[f]), intr).shape[0]
            touched += model.integrate_frame_tensor(dd[f], cc[f], (Rs[f], ts[f]), intr).shape[0]
        e1.record()
        torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    # the same frames through the sync-free pipeline path (fuse_frame_async)
    # on a fresh model: per-frame host syncs gone; the fused model must equal
    # the synchronous one (sorted keys + per-row checksums)
    model2 = GpuVoxelModel(cfg, bucket_count=1 << 21, excess_capacity=1 << 21, device=dev)
    model2._cand_cap = model._cand_cap  # sized by the synchronous run
    for f in range(2):
        model2.fuse_frame_async(dd[f], cc[f], (Rs[f], ts[f]), intr)
    model2.check_async()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for f in range(2, n + 2):
        model2.fuse_frame_async(dd[f], cc[f], (Rs[f], ts[f]), intr)
    a1.record()
    torch.cuda.synchronize()
    ms_async = a0.elapsed_time(a1)
    model2.check_async()

    def digest(m):
        k, pos = m.blocks.snapshot_tensor()
        rows = m.pool[pos.long()].view(torch.int64)
        sums = rows.sum(dim=1)
        kk = k.to(torch.int64) + (1 << 20)
        code = (kk[:, 0] << 42) | (kk[:, 1] << 21) | kk[:, 2]
        order = torch.argsort(code)
        return code[order], sums[order]

    d1, d2 = digest(model), digest(model2)
    same = bool(torch.equal(d1[0], d2[0]) and torch.equal(d1[1], d2[1]))
    return {"workload": f"RC fusion: {n} frames 640x480 inside the 16x3x16 m room, 5 mm voxels, mu 0.06 m",
            "value": n / (ms_async / 1e3), "unit": "frames/s", "ms_per_frame": ms_async / n,
            "path": "GpuVoxelModel.fuse_frame_async (no host sync per frame)",
            "value_sync_api": n / (ms / 1e3), "ms_per_frame_sync_api": ms / n,
            "note_sync_api": "allocate_blocks_tensor + integrate_frame_tensor (reference API: created / touched "
                             "keys returned per frame, host syncs for their counts)",
            "async_equals_sync": same, "wall_s": wall,
            "blocks": model.blocks.approx_size(), "created": created, "touched": touched,
            "integrate_kernel_ms_per_frame": prof.ms["other"] / max(1, prof.count["other"]),
            "gpu_launches": prof.launches}


def cpu_rc_sample():
    """Reference fusion (numpy restatement, 1 thread) on 1 frame of the same workload."""
    from oracle.fusion_oracle import OracleVoxelModel
    from paper_1805_03709_b200 import workloads

    depth, color, Rs, ts, (fx, fy, cx, cy, w, h) = workloads.room_frames(1, 640, 480)
    m = OracleVoxelModel(0.005, 0.06)
    t0 = time.perf_counter()
    m.allocate(depth[0], Rs[0], ts[0], float(fx), float(fy), float(cx), float(cy))
    m.integrate(depth[0], color[0], Rs[0], ts[0], float(fx), float(fy), float(cx), float(cy))
    return 1.0 / (time.perf_counter() - t0)


# ------------------------------------------------------------------ main

def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    from paper_1805_03709_b200 import workloads

    # config 2 (10M keys, 2^22-op batches) on one GPU; config 5 (1e9 keys
    # sharded by hash, 2^24-op batches per GPU) when the job spans N > 1 GPUs
    # or --config5-slice G asks for one GPU's share of a G-GPU run
    c5 = world if world > 1 else args.config5_slice
    if args.live is None:
        args.live = 1_000_000_000 // c5 if c5 > 1 else 10_000_000
    if args.batch_log2 is None:
        args.batch_log2 = 24 if c5 > 1 else 22
    if c5 > 1 and args.steps == 300:
        args.steps = 50  # 2^24-op batches: the pre-generated inputs stay within HBM
    spec = workloads.MixSpec(live=args.live, load_factor=0.7, batch=1 << args.batch_log2, bucket_frac=args.bucket_frac)
    threads = args.cpu_threads or cpu_cores()
    wl = ("config 2: 10M-key block hash set, 50/30/20 insert/find/erase mix, load factor 0.7, "
          f"batches of 2^{args.batch_log2} ops (one launch per batch)") if c5 <= 1 else (
          f"config 5: {spec.live * c5 / 1e9:.2g}B-key block hash set sharded by hash over {c5} GPUs "
          f"({spec.live:,} live keys per GPU), 50/30/20 mix, load factor 0.7, 2^{args.batch_log2}-op batches per GPU"
          + ("" if world > 1 else f"; ONE GPU's slice of a {c5}-GPU run (no routing)"))
    config = {"workload": wl,
              "live_keys_per_gpu": spec.live, "slots_per_gpu": spec.slots, "batch_ops": spec.batch,
              "mix": spec.counts, "key_space": "int3 in [-2^20, 2^20)^3 (injective id map)",
              "l2": f"inputs larger than L2: {spec.slots * 16 / 1e6:.0f} MB table + fresh "
                    f"{spec.batch * 14 / 1e6:.0f} MB batch per step",
              "parallelism": f"hash-sharded x{world}" if world > 1 else "single GPU"}
    if world > 1:
        config["exchange"] = ("peer stores into CUDA-IPC windows over NVLink (csrc/shard.cu)" if args.exchange != "collective"
                              else "NCCL all-to-all (shard.py collective path)")

    if args.impl == "reference":
        # reference arm: the C oracle port of the reference algorithm on host cores
        if rank != 0:
            return
        sys.path.insert(0, str(ROOT))
        times, ok, size = cpu_hash_sample(spec, threads, batches=args.warmup + args.steps)
        t = sum(times[args.warmup:])
        value = args.steps * spec.batch / t / 1e6
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "M ops/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
                "data": "synthetic", "config": config,
                "cpu_baseline": {"value": value, "unit": "M ops/s", "cores": threads, "kind": "port",
                                 "sample": f"{args.steps} mixed batches of {spec.batch} ops on the 10M-key table "
                                           "(C restatement of concurrent_hash.py, bucket-partitioned threads)",
                                 "ok": ok},
                "e2e": {"value": value, "unit": "M ops/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    # VSB_BENCH_ONE_GPU=1: every rank on cuda:0 over gloo -- a functional
    # check of the multi-rank path on a one-GPU box (numbers not meaningful)
    one_gpu = os.environ.get("VSB_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    if world > 1:
        import torch.distributed as dist

        # communicator init lines (rank / nranks) for the launcher's records
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout keeps the one JSON line
        torch.cuda.set_device(local)
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    h = run_hash(args, dev, rank, world)
    if world > 1:  # the route actually used (auto falls back when peer access is unavailable)
        config["exchange"] = ("peer stores into CUDA-IPC windows over NVLink (csrc/shard.cu)"
                              if h.get("exchange") == "peer" else "collective all-to-all (shard.py)")
    def section(fn, *a):
        """A secondary section must never cost the headline line: its failure
        is reported in its own field."""
        try:
            return fn(*a)
        except Exception as exc:  # noqa: BLE001
            import traceback

            traceback.print_exc()
            return {"error": f"{type(exc).__name__}: {exc}"[:300]}

    c1 = None
    if not args.no_config1 and world == 1:
        _free_cuda()
        c1 = section(run_config1, args, dev)
    mc = None
    if not args.no_mc:
        _free_cuda()
        mc = section(run_mc, args, dev, world)
    stream = None
    if not args.no_stream and world == 1:
        _free_cuda()
        stream = section(run_stream, args, dev)
    server = None
    if not args.no_server and world == 1:
        _free_cuda()
        server = section(run_server, args, dev)
    rc = None
    if not args.no_rc and world == 1:
        _free_cuda()
        rc = section(run_rc, args, dev)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        def cpu_hash():
            times, ok, _ = cpu_hash_sample(spec, threads, batches=1)
            return {"value": spec.batch / times[0] / 1e6, "unit": "M ops/s", "cores": threads, "kind": "port",
                    "sample": f"1 mixed batch of {spec.batch} ops on the 10M-key config-2 table (C restatement of "
                              "concurrent_hash.py, bucket-partitioned threads)", "ok": ok}

        def cpu_mc():
            mc_t, mc_n = cpu_mc_sample(threads)
            return {"value": mc_n / mc_t, "unit": "blocks/s", "cores": threads, "kind": "port",
                    "sample": f"{mc_n} room blocks (C restatement of recompute_mc_block)"}

        cpu = section(cpu_hash)
        if not args.no_mc:
            cpu["mc"] = section(cpu_mc)
        if not args.no_rc:
            cpu["rc"] = section(lambda: {"value": cpu_rc_sample(), "unit": "frames/s", "cores": 1, "kind": "port",
                                         "sample": "1 frame 640x480 of the RC workload (numpy restatement of "
                                                   "allocate_blocks + integrate_frame)"})
        if not args.no_stream:
            def cpu_stream():
                v, dt = cpu_stream_baseline(threads, max(args.stream_ticks, STREAM_EVERY))
                return {"value": v, "unit": "M key-ops/s", "cores": min(STREAM_C, threads), "kind": "port",
                        "sample": f"the full config-4 script ({max(args.stream_ticks, STREAM_EVERY)} ticks, 16 clients "
                                  f"incl. fills, reconnects and resets) on the C restatement of BlockHashSet + the "
                                  f"StreamSet FIFO rule, one thread per client, {dt:.1f} s"}

            cpu["stream"] = section(cpu_stream)
    if world > 1:
        import torch.distributed as dist

        oks = torch.tensor([1.0 if h["ok"] else 0.0], device=dev if not one_gpu else "cpu")
        dist.all_reduce(oks, op=dist.ReduceOp.MIN)
        h["ok"] = bool(oks.item() > 0)
    if rank == 0:
        line = {"metric": METRIC, "value": h["value"], "unit": "M ops/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": h["ms_per_step"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic", "config": config,
                "parity_ok": h["ok"], "roofline": h["roofline"], "gpu_launches": h["gpu_launches"],
                "clocks": h["clocks"], "cpu_baseline": cpu, "e2e": h.get("e2e"), "config1": c1, "mc": mc, "stream": stream, "server": server, "rc": rc}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
