"""Aggregate an ncu report's SASS metrics per CUDA source line.

    python scripts/ncu_lines.py gpurun_out/prof_decode.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kern:
    cmd += ["-k", f"regex:{kern}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
agg = {}
src = {}
cur = None
fname = "?"
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ist = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr) - 2:
        continue
    if r[0]:
        cur = (fname, int(r[0])) if r[0].isdigit() else None
        src[cur] = r[1]
        continue
    if cur is None or r[2] in ("...", ""):
        continue
    try:
        a = agg.setdefault(cur, [0, 0])
        a[0] += int(r[ie] or 0)
        a[1] += int(r[ist] or 0)
    except ValueError:
        pass
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total instructions {ti}, stall samples {ts}")
for ln, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{ln[0][:14]:>14}:{ln[1]:<4d} inst {100*i/ti:5.1f}%  stall {100*s/ts:5.1f}%  {src.get(ln, '')[:90]}")
