# quick iteration: parity subset + bench variants
set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "not full_size" > gpurun_out/par.log 2>&1; echo rc=$?
tail -3 gpurun_out/par.log
for mb in 2 3 4; do
THERMO_DECODE_MINB=$mb timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_mb$mb.json 2> gpurun_out/bench_mb$mb.err; echo rc=$?
done
