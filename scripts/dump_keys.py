"""One ingest + build of a bench workload with THERMO_DUMP_KEYS set: writes the
retained keys for scripts/cub_sort.cu (measurement only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
w, path = sys.argv[1], sys.argv[2]
os.environ["THERMO_DUMP_KEYS"] = path
import bench  # noqa: E402
from paper_2507_18729_b200 import BOTH, Thermo  # noqa: E402

t = bench.make_trace(w, "cuda")
th = Thermo(max_launches=max(1, int(t.meta.get("launches", 1))),
            max_warps_per_launch=max(1, int(t.meta.get("warps", 1 << 20))), max_pcs=int(t.meta.get("pcs", 256)))
th.register_objects(t.objects)
th.ingest(t.records)
th.build(BOTH)
print(w, th.stats()["keys_emitted"])
