"""Summaries of scripts/gpu_ncu_more.sh captures into profiles/<tag>_ncu_<name>.txt
(run here after the GPU call)."""
import pathlib
import subprocess
import sys

sys.path.insert(0, str(pathlib.Path(__file__).parent))
from ncu_summary import KEYS, stalls

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
EXTRA = ["l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
         "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum"]


def raw_all(rep):
    import csv

    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    return [(v[h.index("Kernel Name")], {n: (v[i], u[i]) for i, n in enumerate(h)}) for v in r[2:]]


for name, rep, cmd in [("stream", "gpurun_out/prof_stream.ncu-rep", "k_multi_insert (config-4 fan-out insert)"),
                       ("rc", "gpurun_out/prof_rc.ncu-rep", "k_rc_integrate (RC fusion)"),
                       ("shard", "gpurun_out/prof_shard.ncu-rep", "peer-shard kernels at world 1")]:
    if not pathlib.Path(rep).exists():
        print("missing", rep)
        continue
    lines = [f"# ncu --set full summary ({tag}): {cmd}, from {rep.split('/')[-1]}",
             "# command: scripts/gpu_ncu_more.sh"]
    for kname, d in raw_all(rep):
        lines.append(f"## {kname[:110]}")
        for k in KEYS + EXTRA:
            if k in d:
                lines.append(f"{k:60s} {d[k][0]} {d[k][1]}")
    lines.append("# top stall-sampled source lines (share of warp stall samples, all captured launches)")
    for s, p, f, l, src in stalls(rep, 15):
        lines.append(f"{s:7d} {p:5.1f}% {f}:{l} {src[:100]}")
    pathlib.Path(f"profiles/{tag}_ncu_{name}.txt").write_text("\n".join(lines) + "\n")
    print("\n".join(lines[:14]))
