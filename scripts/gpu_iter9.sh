# parity + benches after the vectorised histogram / indicator sweeps
set -x
timeout 1200 python -m pytest tests -x -q -m gpu --timeout 600 > gpurun_out/par_full.log 2>&1; echo rc=$?
tail -15 gpurun_out/par_full.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; python -c "import json;d=json.load(open('gpurun_out/bench_q.json'));print(d['ms_per_step'], d['phase_ms'])"
timeout 300 python bench.py --workload stencil --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_st.json 2>gpurun_out/bench_st.err; python -c "import json;d=json.load(open('gpurun_out/bench_st.json'));print('stencil', d['ms_per_step'], d['phase_ms'])"
timeout 600 python bench.py --workload synthetic --steps 5 --warmup 3 --no-e2e --dedup segment --no-cpu-baseline > gpurun_out/bench_synth_seg.json 2>gpurun_out/bench_synth_seg.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_synth_seg.json'));print('seg', d['value'], d['ms_per_step'], d['phase_ms'])"
timeout 900 python bench.py --workload spmv --steps 2 --warmup 3 --no-e2e --dedup segment --no-cpu-baseline > gpurun_out/bench_spmv_seg.json 2>gpurun_out/bench_spmv_seg.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_spmv_seg.json'));print('spmv seg', d['value'], d['ms_per_step'], d['phase_ms'])"
