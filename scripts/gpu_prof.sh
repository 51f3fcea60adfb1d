# parity + bench variants + decode profile after a change
set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "not full_size" > gpurun_out/par.log 2>&1; echo rc=$?
tail -2 gpurun_out/par.log
for mb in 2 3; do
THERMO_DECODE_MINB=$mb timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_mb$mb.json 2> gpurun_out/bench_mb$mb.err; echo rc=$?
done
THERMO_DECODE_MINB=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -o gpurun_out/prof_decode4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_decode3.log 2>&1; echo rc=$?
