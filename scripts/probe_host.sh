free -g; nproc; cat /proc/cpuinfo | grep "model name" | head -1
python - <<'PY'
import time, sys
sys.path.insert(0, '.')
import torch, oracle, tracegen as tg
t0 = time.time(); t = tg.stencil(8192, device="cuda"); torch.cuda.synchronize(); print("gen", time.time() - t0)
recs = t.records.cpu(); print("copy", time.time() - t0)
o = oracle.Oracle([x[:4] for x in t.objects])
t1 = time.time()
for a in range(0, recs.shape[0], 1 << 25):
    o.ingest(recs[a:a + (1 << 25)])
print("ingest", time.time() - t1)
o.build(); print("build", time.time() - t1)
ind = o.classify(); print("classify", time.time() - t1, ind[0]["labels"])
import resource; print("maxrss GB", resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6)
PY
