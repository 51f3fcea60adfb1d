# parity + bench (minb 2/3/4) + ncu of the decode kernel
set -x
timeout 300 python -m pytest tests -x -q -m gpu --timeout 120 > gpurun_out/par.log 2>&1; echo rc=$?
tail -5 gpurun_out/par.log
for mb in 2 3 4; do
THERMO_DECODE_MINB=$mb timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_mb$mb.json 2> gpurun_out/bench_mb$mb.err; echo rc=$?
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|decode_general|seg_chunk" -s 6 -c 3 -o gpurun_out/prof_v8 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_v8.log 2>&1; echo rc=$?
