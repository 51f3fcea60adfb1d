"""Per-kernel summary metrics from an ncu --set full report (raw page) as JSON.

    python scripts/ncu_metrics.py gpurun_out/prof_full.ncu-rep > profiles/r1_ncu_full_metrics.json
"""
import csv
import io
import json
import subprocess
import sys

WANT = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers"]
STALL = "smsp__pcsamp_warps_issue_stalled_"
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
res = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    e = {"kernel": d.get("Kernel Name", "?")}
    for k in WANT:
        if k in d:
            try:
                v = float(d[k].replace(",", ""))
                u = dict(zip(hdr, units)).get(k, "")
                if u in ("Kbyte", "KB"): v *= 1e3
                elif u in ("Mbyte", "MB"): v *= 1e6
                elif u in ("Gbyte", "GB"): v *= 1e9
                elif u in ("usecond", "us"): v *= 1e3
                elif u in ("msecond", "ms"): v *= 1e6
                e[k] = v
            except ValueError:
                pass
    for k, v in d.items():
        if k.startswith(STALL) and not k.endswith("_not_issued") and v.replace(",", "").isdigit() and int(v.replace(",", "")) > 500:
            e[k] = int(v.replace(",", ""))
    res.append(e)
print(json.dumps(res, indent=1))
