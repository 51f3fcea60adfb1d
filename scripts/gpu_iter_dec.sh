# decode iteration: parity subset, SGEMM bench x2, stencil launch list, decode ncu capture with source
set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "small_workloads or random_traces or many_objects or window or warp_records or synthetic_medium or hot_sector or access_counts or sampled_block or gemm_full" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -2 gpurun_out/q_pytest.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_bench_$i.json 2> gpurun_out/q_bench.err; echo rc=$?; done
timeout 300 python bench.py --workload spmv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_spmv.json 2> gpurun_out/q_spmv.err; echo rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"thermo::" --csv --log-file gpurun_out/launches_stencil.csv python bench.py --workload stencil --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_stencil.log 2>&1; echo rc=$?
timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::decode_kernel" -s 3 -c 1 -o gpurun_out/prof_dec python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_dec.log 2>&1; echo rc=$?
python - <<'PY'
import json
for f in ["q_bench_1", "q_bench_2", "q_spmv"]:
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, "ms/step %.3f" % d["ms_per_step"], {k: round(v, 3) for k, v in d["phase_ms"].items()}, "frac %.3f" % d["roofline"]["frac"])
    except Exception as e:
        print(f, "ERR", e)
PY
