# full GPU parity suite, smoke and a quick bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 > gpurun_out/par_full.log 2>&1; echo rc=$?
tail -5 gpurun_out/par_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$?
tail -2 gpurun_out/smoke.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo rc=$?
cat gpurun_out/bench_q.json
cat MEASURED_PEAKS.json 2>/dev/null
