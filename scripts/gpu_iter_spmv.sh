# SpMV decode variants + quick parity
set -x
timeout 600 python -m pytest tests -x -q -m gpu -k "small_workloads or random_traces or hot_sector or warp_records or synthetic_medium" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -2 gpurun_out/q_pytest.log
for v in 1; do timeout 300 python bench.py --workload spmv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_spmv_$v.json 2> gpurun_out/q_spmv_$v.err; echo rc=$?; done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"thermo::" --csv --log-file gpurun_out/launches_spmv.csv python bench.py --workload spmv --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_spmv.log 2>&1; echo rc=$?
python - <<'PY'
import json
for f in ["q_bench", "q_spmv_2", "q_spmv_4"]:
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, "ms/step %.3f" % d["ms_per_step"], {k: round(v, 3) for k, v in d["phase_ms"].items()}, "frac %.3f" % d["roofline"]["frac"])
    except Exception as e:
        print(f, "ERR", e)
PY
