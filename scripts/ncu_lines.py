"""Per-source-line stall samples and executed instructions of one kernel in an ncu report.
  python scripts/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f = None
res = []
tot_s = tot_i = 0
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit() and r[2] == "-":
        try:
            s, i = int(r[4]), int(r[7])
        except ValueError:
            continue
        res.append((s, i, f, int(r[0]), r[1].strip()))
        tot_s += s
        tot_i += i
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, i, f, l, src in sorted(res, reverse=True)[:n]:
    print(f"{100*s/max(tot_s,1):5.1f}% {100*i/max(tot_i,1):5.1f}%i  {f}:{l}  {src[:100]}")
