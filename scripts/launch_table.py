"""Per-kernel time / DRAM bytes per launch and share from an ncu launch-list CSV
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = d["Kernel Name"].split("(")[0][:44]
    m = d["Metric Name"]
    data[k][m] += float(d["Metric Value"].replace(",", ""))
    if m == "gpu__time_duration.sum":
        cnt[k] += 1
tot = sum(v["gpu__time_duration.sum"] for v in data.values())
for k, v in sorted(data.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    t = v["gpu__time_duration.sum"]
    b = v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
    print(f"{k:44s} n={cnt[k]:3d} ms/launch={t / cnt[k] / 1e6:8.3f} share={t / tot:6.3f} "
          f"GB/launch={b / cnt[k] / 1e9:6.2f} GB/s={b / t:7.0f}")
