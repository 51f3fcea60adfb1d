# parity with the batch decode + bench batch vs warp decode + ncu of the batch kernel
set -x
export THERMO_DECODE=${THERMO_DECODE:-b}
timeout 300 python -m pytest tests -x -q -m gpu --timeout 120 > gpurun_out/par.log 2>&1; echo rc=$?
tail -5 gpurun_out/par.log
timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err; echo rc=$?
THERMO_DECODE=w timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_warp.json 2> gpurun_out/bench_warp.err; echo rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"decode_batch|decode_general" -s 4 -c 2 -o gpurun_out/prof_batch python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_batch.log 2>&1; echo rc=$?
