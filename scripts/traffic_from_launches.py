"""DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per launch of each
library kernel, from ncu launch lists (scripts/gpu_r2_launch.sh), as the
`roofline.traffic` table bench.py reads: profiles/r2_traffic.json =
{workload: {kernel: bytes per launch}}.

    python scripts/traffic_from_launches.py spmv=gpurun_out/ll_spmv.csv sgemm=... > profiles/r2_traffic.json
"""
import collections
import csv
import json
import sys

NAMES = ("decode_kernel", "decode_lane_kernel", "decode_warp_kernel", "decode_general_kernel", "seg_coarse_kernel",
         "seg_fine_kernel", "seg_chunk_kernel", "seg_big_kernel", "seg_big_pc_kernel", "object_hist_kernel")
out = {}
for arg in sys.argv[1:]:
    w, path = arg.split("=", 1)
    rows = list(csv.reader(open(path)))
    hdr = None
    byt, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        base = d["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0].strip()
        if base not in NAMES:
            continue
        m = d["Metric Name"]
        v = float(d["Metric Value"].replace(",", ""))
        if m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            byt[base] += v
        elif m == "gpu__time_duration.sum":
            cnt[base] += 1
    out[w] = {k: byt[k] / cnt[k] for k in cnt}
print(json.dumps(out, indent=1))
