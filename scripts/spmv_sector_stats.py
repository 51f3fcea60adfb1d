"""Per-sector key statistics of the SpMV s=24 trace (distinct (sector, warp)
pairs per sector, records per sector) -- sizing data for the count phase."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import tracegen as tg

t = tg.spmv(int(sys.argv[1]) if len(sys.argv) > 1 else 24, 16, device="cuda")
r = t.records.to(torch.int64) & 0xFFFFFFFF
addr = r[:, 0] | ((r[:, 1] & 0xFFFF) << 32)
warp = r[:, 2]
del r
bases = torch.tensor(sorted(o[0] for o in t.objects), device="cuda")
lens = {o[0]: o[1] for o in t.objects}
soff, acc = [], 0
for b in bases.tolist():
    soff.append(acc); acc += (lens[b] + 31) // 32
soff = torch.tensor(soff, device="cuda")
oi = torch.searchsorted(bases, addr, right=True) - 1
g = soff[oi] + (addr - bases[oi]) // 32
del addr, oi
out = {"records": int(g.shape[0]), "S_tot": acc}
rec_per = torch.bincount(g, minlength=acc)
pair = torch.unique(g * (1 << 20) + warp)
gp = pair >> 20
dist_per = torch.bincount(gp, minlength=acc)
out["distinct_pairs"] = int(pair.shape[0])
for name, c in (("records_per_sector", rec_per), ("distinct_per_sector", dist_per)):
    d = {}
    for th in (256, 1024, 2048, 4096, 8192, 16384, 65536):
        m = c >= th
        d[str(th)] = {"sectors": int(m.sum()), "items": int(c[m].sum())}
    d["max"] = int(c.max())
    out[name] = d
print(json.dumps(out, indent=1))
