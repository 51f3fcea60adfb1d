"""Per-kernel totals of an ncu launch list (gpu__time_duration.sum CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k[:50]:50s} n={len(v):3d} mean_us={sum(v) / len(v) / 1e3:10.1f} share={100 * sum(v) / tot:5.1f}%")
