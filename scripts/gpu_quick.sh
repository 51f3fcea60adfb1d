# parity + one bench line (fast iteration)
set -x
timeout 300 python -m pytest tests -x -q -m gpu -k "not full_size" --timeout 120 > gpurun_out/par.log 2>&1; echo rc=$?
tail -3 gpurun_out/par.log
timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo rc=$?
