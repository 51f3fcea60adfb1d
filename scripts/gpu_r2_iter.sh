# iteration: GPU parity subset (or all with FULL=1) + bench lines of the 4 configs with stats
set -x
if [ "${FULL:-0}" = "1" ]; then
  timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/it_pytest.log 2>&1; echo rc=$?
else
  timeout 900 python -m pytest tests -x -q -m gpu -k "${K:-small_workloads or random_traces or random_hot or hot_sector or warp_records or synthetic_medium or shards or empty}" > gpurun_out/it_pytest.log 2>&1; echo rc=$?
fi
tail -3 gpurun_out/it_pytest.log
grep -E "Error|assert|FAILED" gpurun_out/it_pytest.log | head -20
for w in ${WL:-sgemm stencil spmv}; do timeout 600 python bench.py --workload $w --only --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/it_bench_$w.json 2> gpurun_out/it_bench_$w.err; echo rc=$?; tail -2 gpurun_out/it_bench_$w.err; done
python - <<'PY'
import json
for w in ["sgemm", "stencil", "spmv", "synthetic"]:
    try:
        d = json.load(open(f"gpurun_out/it_bench_{w}.json"))
        print(w, "ms/step %.2f" % d["ms_per_step"], "Grec/s %.2f" % (d["value"] / 1e9), {k: round(v, 2) for k, v in d["phase_ms"].items()}, d["stats"])
    except Exception as e:
        print(w, "ERR", e)
PY
