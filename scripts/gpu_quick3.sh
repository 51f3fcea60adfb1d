set -x
timeout 300 python -m pytest tests -x -q -m gpu --timeout 120 > gpurun_out/par.log 2>&1; echo rc=$?
tail -3 gpurun_out/par.log
for mb in 2 3 4; do
THERMO_DECODE_MINB=$mb timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_mb$mb.json 2> gpurun_out/bench_mb$mb.err; echo rc=$?
done
