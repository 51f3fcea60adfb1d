# quick iteration: decode-path parity subset + default bench lines (SGEMM lane and warp formats)
set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "small_workloads or random_traces or many_objects or window or warp_records or synthetic_medium or hot_sector or access_counts or sampled_block" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -2 gpurun_out/q_pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo rc=$?
timeout 300 python bench.py --format warp --no-cpu-baseline --no-e2e > gpurun_out/q_bench_warp.json 2> gpurun_out/q_bench_warp.err; echo rc=$?
python - <<'PY'
import json
for f in ["q_bench", "q_bench_warp"]:
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, "ms/step %.3f" % d["ms_per_step"], {k: round(v, 3) for k, v in d["phase_ms"].items()}, "frac %.3f" % d["roofline"]["frac"])
    except Exception as e:
        print(f, "ERR", e)
PY
