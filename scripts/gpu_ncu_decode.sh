set -x
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel" -s 2 -c 1 -o gpurun_out/prof_dec python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_dec.log 2>&1; echo rc=$?
