# parity + A/B: hash-set chunk kernel; decode occupancy 3 vs 4 blocks/SM
set -x
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/par_full.log 2>&1; echo rc=$?
tail -5 gpurun_out/par_full.log
for m in 3 4 3 4; do THERMO_DEC_MINB=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_m$m.json 2>gpurun_out/bench_m$m.err; python -c "import json;d=json.load(open('gpurun_out/bench_m$m.json'));print($m, d['ms_per_step'], d['phase_ms'])"; done
timeout 300 python bench.py --workload stencil --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_st.json 2>gpurun_out/bench_st.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_st.json'));print('stencil', d['ms_per_step'], d['phase_ms'])"
