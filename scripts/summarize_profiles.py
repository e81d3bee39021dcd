"""Turn the ncu captures of scripts/gpu_bench.sh (gpurun_out/) into the
committed summaries under profiles/ (run here, after the GPU call)."""
import collections, csv, json, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).parent))
from ncu_summary import KEYS, raw, stalls

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = {}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for name, rep, kern in [("apply", "gpurun_out/prof_apply.ncu-rep", "k_apply"),
                        ("mc", "gpurun_out/prof_mc.ncu-rep", "k_mc_encode")]:
    d = raw(rep)
    lines = [f"# ncu --set full summary: vsb::{kern} ({tag}), from {rep.split('/')[-1]}",
             f"# command: scripts/gpu_bench.sh (ncu --set full --clock-control none --import-source on -k regex:{kern} -s N -c 1)"]
    for k in KEYS + ["l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
                     "lts__t_requests_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
                     "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum"]:
        if k in d:
            lines.append(f"{k:60s} {d[k][0]} {d[k][1]}")
    lines.append("# top stall-sampled source lines (share of warp stall samples)")
    for s, p, f, l, src in stalls(rep, 20):
        lines.append(f"{s:7d} {p:5.1f}% {f}:{l} {src[:100]}")
    pathlib.Path(f"profiles/{tag}_ncu_{name}.txt").write_text("\n".join(lines) + "\n")
    rd = float(d["dram__bytes_read.sum"][0]) * UNITS[d["dram__bytes_read.sum"][1]]
    wr = float(d["dram__bytes_write.sum"][0]) * UNITS[d["dram__bytes_write.sum"][1]]
    out[kern] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                 "ncu_duration": " ".join(d["gpu__time_duration.sum"]), "source": f"profiles/{tag}_ncu_{name}.txt"}
pathlib.Path("profiles/ncu_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
rows = [r for r in csv.reader(open("gpurun_out/launches.csv")) if r]
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h, start = r, i + 1
        break
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[start:]:
    name = r[ik].split("(")[0]
    agg.setdefault(name, [0, 0.0])
    agg[name][0] += 1
    agg[name][1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
lines = [f"# ncu launch list ({tag}): ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_",
         "#   python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --mc-steps 2 --stream-ticks 20   (cold-cache, serialised)",
         f"{'kernel':40s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>10s} {'share':>7s}"]
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"{k:40s} {c:8d} {v / 1e6:10.3f} {v / c / 1e3:10.1f} {100 * v / tot:6.1f}%")
pathlib.Path(f"profiles/{tag}_launches.txt").write_text("\n".join(lines) + "\n")
print("\n".join(lines[:12]))
print(json.dumps(out, indent=1))
