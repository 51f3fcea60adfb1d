# parity + benches + decode profile, with short timeouts (a hang costs minutes, not the budget)
set -x
timeout 300 python -m pytest tests -x -q -m gpu -k "not full_size" --timeout 60 > gpurun_out/par.log 2>&1; echo rc=$?
tail -3 gpurun_out/par.log
for mb in 2 3; do
THERMO_DECODE_MINB=$mb timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_mb$mb.json 2> gpurun_out/bench_mb$mb.err; echo rc=$?
done
timeout 120 python bench.py --steps 5 --warmup 3 --dedup sort --no-cpu-baseline --no-e2e > gpurun_out/bench_sort.json 2> gpurun_out/bench_sort.err; echo rc=$?
THERMO_DECODE_MINB=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|seg_chunk" -s 6 -c 2 -o gpurun_out/prof_it python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_it.log 2>&1; echo rc=$?
