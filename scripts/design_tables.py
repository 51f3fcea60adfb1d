"""Markdown tables for DESIGN.md §5 / §8 from the committed evidence:
profiles/r2_bench_default.json (bench line, every config) and
profiles/r2_traffic.json (ncu DRAM bytes per launch).

    python scripts/design_tables.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
b = json.load(open(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r2_bench_default.json")))
traffic = json.load(open(os.path.join(ROOT, "profiles", "r2_traffic.json")))

ROW = {"decode_kernel": "a2+a3", "decode_lane_kernel": "a2+a3", "decode_general_kernel": "a2+a3", "seg_scan": "a4",
       "seg_coarse_kernel": "a4", "seg_fine_kernel": "a4", "seg_chunk_kernel": "a4+a5+a6(pc)",
       "seg_big_kernel": "a4+a5+a6(pc)", "object_hist_kernel": "a6", "indicator_kernels": "a7"}
BYTES = {"decode_kernel": "16 B × records", "decode_lane_kernel": "16 B × records",
         "seg_coarse_kernel": "16 B × keys", "seg_fine_kernel": "16 B × keys",
         "seg_chunk_kernel": "8 B × keys + 36 B × touched sectors", "object_hist_kernel": "36 B × sectors",
         "indicator_kernels": "72 B × sectors (two tile passes)"}
BOUND = {"decode_kernel": "HBM read (issue-bound, §8)", "decode_lane_kernel": "HBM read (issue-bound, §8)",
         "decode_general_kernel": "L2 / issue", "seg_scan": "HBM", "seg_coarse_kernel": "HBM (smem atomics, §8)",
         "seg_fine_kernel": "HBM (smem atomics, §8)", "seg_chunk_kernel": "smem atomics",
         "seg_big_kernel": "smem atomics / L2", "object_hist_kernel": "HBM", "indicator_kernels": "HBM"}

print("KERNEL_TABLE (SpMV)\n")
print("| Kernel | Row | Roofline | Algorithmic bytes per launch | SpMV ms | frac of peak | ncu DRAM / launch |")
print("|---|---|---|---|---|---|---|")
tr = traffic.get("spmv", {})
for k, v in b["kernels"].items():
    t = tr.get(k)
    if k == "seg_big_kernel" and "seg_big_pc_kernel" in tr:
        t = (tr.get(k, 0) or 0) + tr["seg_big_pc_kernel"]
    frac = f"{v['frac']:.3f}" if "frac" in v else "—"
    print(f"| `{k}` | {ROW.get(k, '')} | {BOUND.get(k, '')} | {BYTES.get(k, '—')} | {v['ms_per_launch']:.2f} | {frac} | "
          f"{'%.2f GB' % (t / 1e9) if t else '—'} |")

print("\nBENCH_TABLE\n")
print("| config | records | keys | ms / step | G records/s | dominant kernel (frac of HBM) | pipeline frac | e2e |")
print("|---|---|---|---|---|---|---|---|")


def line(name, d, head):
    r = d["roofline"]
    e2e = d.get("e2e")
    e = f"{e2e['value'] / 1e9:.2f} G/s ({e2e['h2d_bytes_per_step'] / 1e9:.2f} GB H2D per step)" if head and e2e else "—"
    rec = d.get("records") or d["config"]["records"]
    bold = "**" if head else ""
    print(f"| {bold}{name}{bold} | {rec / 1e6:.1f} M | {d['stats']['keys_emitted'] / 1e6:.1f} M | {bold}{d['ms_per_step']:.2f}{bold} | "
          f"{bold}{d['value'] / 1e9:.2f}{bold} | {r['kernel']} {r['ms_per_launch']:.2f} ms ({r['frac']:.3f}) | "
          f"{d['pipeline_roofline']['frac']:.3f} | {e} |")


line("SpMV R-MAT s=24", b, True)
names = {"sgemm": "SGEMM 1024², K=128", "stencil": "stencil 8192²", "synthetic": "synthetic slice"}
for k, d in b.get("configs", {}).items():
    line(names.get(k, k), d, False)

print("\nKERNEL_SPLIT\n")
print(", ".join(f"{k} {v['ms_per_launch']:.2f}" for k, v in b["kernels"].items()) +
      f"; other (resets, memsets, host syncs) {b['ms_per_step'] - sum(v['ms_per_launch'] for v in b['kernels'].values()):.2f}")
