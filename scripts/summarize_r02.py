"""Summaries of the round-2 ncu captures (scripts/gpu_r02_ncu.sh) into
profiles/r02_ncu_<name>.txt and the launch list into profiles/r02_launches.txt
(run here after the GPU call)."""
import csv
import pathlib
import subprocess
import sys

sys.path.insert(0, str(pathlib.Path(__file__).parent))
from ncu_summary import KEYS  # noqa: E402

EXTRA = ["dram__sectors_read.sum", "dram__sectors_write.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
         "lts__t_sectors_srcunit_tex_op_red.sum", "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
         "sm__cycles_elapsed.avg.per_second"]
CAPS = [("apply", "r02_apply", "k_apply (config 2, one 2^22-op mixed batch)"),
        ("mc", "r02_mc", "k_mc_encode<1,0,0> (config 3 full encode, 2,080,160 blocks)"),
        ("mcaux", "r02_mcaux", "k_mc_faces / k_mc_compact (config 3 incremental packs, two-pass compaction)"),
        ("stream", "r02_stream", "config-4 tick kernels: k_dedup_small, k_multi_fan_small, k_multi_extract"),
        ("server", "r02_server", "SURVEY 3.1 on_tsdf_batch kernels (6 launches per tick): k_dedup_small, k_insert_t (MC map; TSDF put with its latest-write claims), k_put_rows, k_mc_encode<1,1,0,0> (faces, out_rows, FRESH settle), k_multi_fan_small"),
        ("rc", "r02_rc", "RC fusion: k_rc_cull_table, k_rc_integrate"),
        ("shard", "r02_shard", "peer-shard route at world 1, config-5 slice (125M keys, 2^24-op batches, 16 bucket regions): "
                            "k_wpart_count, k_wpart_base, k_wpart_push, k_shard_apply, k_shard_return")]


def raw_all(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    return [(v[h.index("Kernel Name")], {n: (v[i], u[i]) for i, n in enumerate(h)}) for v in r[2:]]


def stalls(rep, kernel, n=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", kernel], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    f, res = None, []
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) > 4 and r[0].isdigit() and r[2] == "-":
            try:
                res.append((int(r[4]), f, int(r[0]), r[1].strip()))
            except ValueError:
                pass
    tot = sum(x[0] for x in res) or 1
    return [(s, 100 * s / tot, f, l, src) for s, f, l, src in sorted(res, reverse=True)[:n]]


def main(src="gpurun_out", tag="r02", only=""):
    for name, rep, what in CAPS:
        if only and name not in only.split(","):
            continue
        path = f"{src}/{rep}.ncu-rep"
        if not pathlib.Path(path).exists():
            print("missing", path)
            continue
        lines = [f"# ncu --set full --clock-control none summary ({tag}): {what}",
                 f"# from {rep}.ncu-rep, command in scripts/gpu_r02_ncu.sh"
                 + (" (re-captured after the late changes)" if name in ("shard", "server") else "")]
        seen = set()
        for kname, d in raw_all(path):
            lines.append(f"## {kname[:120]}")
            for k in KEYS + EXTRA:
                if k in d:
                    lines.append(f"{k:60s} {d[k][0]} {d[k][1]}")
            short = kname.split("(")[0].split("<")[0].split("::")[-1]
            if short in seen:
                continue
            seen.add(short)
            lines.append(f"# top stall-sampled source lines of {short} (share of its warp stall samples)")
            for s, p, f, l, code in stalls(path, short):
                lines.append(f"{s:7d} {p:5.1f}% {f}:{l} {code[:100]}")
        pathlib.Path(f"profiles/{tag}_ncu_{name}.txt").write_text("\n".join(lines) + "\n")
        print("wrote", f"profiles/{tag}_ncu_{name}.txt")
    if pathlib.Path(f"{src}/launches.csv").exists():
        out = subprocess.run([sys.executable, "scripts/launch_summary.py", f"{src}/launches.csv"], capture_output=True,
                             text=True).stdout
        pathlib.Path(f"profiles/{tag}_launches.txt").write_text(
            "# ncu --metrics gpu__time_duration.sum --clock-control none launch list of\n"
            "# python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-mc-parity --mc-steps 2 --stream-ticks 20 "
            "--rc-frames 3\n# (per-launch times are cold-cache and serialised: compare shares, not absolutes)\n" + out)
        print("wrote", f"profiles/{tag}_launches.txt")


if __name__ == "__main__":
    main(*sys.argv[1:])
