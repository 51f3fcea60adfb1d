"""Sampled-block mode on the full SGEMM trace (BJ configs[1], 270.5 M records,
block 0 of 32 warps): ingest + build with the DENSE warp-bitmask path vs SEGMENT,
CUDA events on the context's stream.  python scripts/dense_timing.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen as tg  # noqa: E402
from paper_2507_18729_b200 import BOTH, Thermo  # noqa: E402

t = tg.gemm(1024, 1024, 128, "v00", device="cuda")
out = {}
for name, dedup in (("dense", 4), ("segment", 3)):
    stream = torch.cuda.current_stream()
    th = Thermo(max_launches=1, max_warps_per_launch=1 << 15, max_pcs=256, block_warps=32, block_id=0,
                dedup=dedup, stream=stream.cuda_stream)
    th.register_objects(t.objects)
    for _ in range(3):
        th.reset(); th.ingest(t.records); th.build(BOTH)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(10):
        th.reset(); th.ingest(t.records); th.build(BOTH)
    e1.record(stream)
    torch.cuda.synchronize()
    st = th.stats()
    out[name] = {"ms_per_step": e0.elapsed_time(e1) / 10, "ms_decode": st["ms_decode"], "ms_dedup": st["ms_dedup"],
                 "ms_count": st["ms_count"], "keys": st["keys_emitted"], "distinct_pairs": st["distinct_pairs"],
                 "dedup_used": st["dedup_used"]}
    th.close()
print(json.dumps(out))
