# quick iteration on every workload: decode/count parity subset, full-size tests, bench lines
set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "small_workloads or random_traces or many_objects or window or warp_records or synthetic_medium or hot_sector or access_counts or sampled_block or full_size or shards" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -2 gpurun_out/q_pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo rc=$?
for w in stencil spmv synthetic; do timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err; echo rc=$?; done
python - <<'PY'
import json
for f in ["q_bench", "q_stencil", "q_spmv", "q_synthetic"]:
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, "ms/step %.3f" % d["ms_per_step"], {k: round(v, 3) for k, v in d["phase_ms"].items()}, "frac %.3f" % d["roofline"]["frac"])
    except Exception as e:
        print(f, "ERR", e)
PY
