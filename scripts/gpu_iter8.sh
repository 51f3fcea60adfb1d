# parity + sgemm/stencil bench with the warp-aggregated scatter
set -x
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/par_full.log 2>&1; echo rc=$?
tail -3 gpurun_out/par_full.log
for w in sgemm sgemm; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; python -c "import json;d=json.load(open('gpurun_out/bench_q.json'));print(d['ms_per_step'], d['phase_ms'])"; done
timeout 300 python bench.py --workload stencil --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_st.json 2>gpurun_out/bench_st.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_st.json'));print('stencil', d['ms_per_step'], d['phase_ms'])"
timeout 600 python bench.py --workload spmv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_spmv.json 2> gpurun_out/bench_spmv.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_spmv.json'));print('spmv', d['ms_per_step'], d['phase_ms'], d['config'])"
