"""Per-kernel mean/max durations from an ncu --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
d = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        if x["Metric Name"] == "gpu__time_duration.sum":
            d[x["Kernel Name"][:70]].append(float(x["Metric Value"].replace(",", "")))
for k, v in d.items():
    print(f"{k:70s} n={len(v):4d} mean={sum(v) / len(v) / 1000:8.1f}us max={max(v) / 1000:8.1f}us")
