"""Where the decoder's pre-dedup leaves duplicate keys (measurement only).

    python scripts/key_redundancy.py spmv      # on a GPU box

One ingest + build of a bench workload with THERMO_DUMP_KEYS set, then, per
object: keys emitted, distinct (sector, launch, warp, pc) keys (the best a
decoder-side pre-dedup could reach) and distinct (sector, launch, warp) pairs.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
w = sys.argv[1]
path = f"/tmp/keys_{w}.bin"
os.environ["THERMO_DUMP_KEYS"] = path
import bench  # noqa: E402
from paper_2507_18729_b200 import BOTH, Thermo  # noqa: E402

t = bench.make_trace(w, "cuda")
ml = max(1, int(t.meta.get("launches", 1)))
mw = max(1, int(t.meta.get("warps", 1 << 20)))
mp = int(t.meta.get("pcs", 256))
th = Thermo(max_launches=ml, max_warps_per_launch=mw, max_pcs=mp)
th.register_objects(t.objects)
th.ingest(t.records)
th.build(BOTH)
st = th.stats()
th.close()
del t.records
torch.cuda.empty_cache()

hdr = np.fromfile(path, dtype=np.uint64, count=2)
n, width = int(hdr[0]), int(hdr[1])
keys = torch.from_numpy(np.fromfile(path, dtype=np.int64, offset=16, count=n)).cuda()
L, W, P = (ml - 1).bit_length(), (mw - 1).bit_length(), (mp - 1).bit_length()
S = width - L - W - P
objs = sorted(t.objects, key=lambda o: (o[2] << 48) | o[0])
soff, names = [0], []
for o in objs:
    soff.append(soff[-1] + (o[1] + 31) // 32)
    names.append(o[4] if len(o) > 4 else str(o[3]))
pre = keys >> 8  # [g][launch][warp][pc]
g = (pre >> (L + W + P)) & ((1 << S) - 1)
bounds = torch.tensor(soff[1:], device="cuda")
oid = torch.bucketize(g, bounds, right=True)
res = {"workload": w, "keys": n, "stats": {k: st[k] for k in ("keys_emitted", "distinct_pairs", "distinct_pc_pairs")},
       "objects": []}
for k, nm in enumerate(names):
    sel = pre[oid == k]
    if sel.numel() == 0:
        continue
    d_full = torch.unique(sel).numel()
    d_pair = torch.unique(sel >> P).numel()
    res["objects"].append({"object": nm, "keys": int(sel.numel()), "distinct_sector_launch_warp_pc": d_full,
                           "distinct_sector_launch_warp": d_pair})
    del sel
print(json.dumps(res, indent=1))

# SEGMENT's big sectors (>= 2048 keys): keys, passes of 6144, re-read volume
cnt = torch.bincount(g, minlength=soff[-1])
big = cnt[cnt >= 2048].to(torch.int64)
passes = (big + 6143) // 6144
rest = cnt[(cnt > 0) & (cnt < 2048)].to(torch.int64)
print(json.dumps({"big_sectors": int(big.numel()), "big_keys": int(big.sum()), "big_key_reads": int((big * passes).sum()),
                  "big_passes": int(passes.sum()), "max_keys": int(big.max()) if big.numel() else 0,
                  "normal_sectors": int(rest.numel()), "normal_keys": int(rest.sum()),
                  "normal_hist_log2": torch.bincount(torch.log2(rest.float()).long()).tolist()}))
