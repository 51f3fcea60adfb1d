# one full ncu capture (with source) of the fast decode kernel and the chunk kernel
set -x
timeout 500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::(decode_kernel|seg_chunk_kernel)" -s 2 -c 2 -o gpurun_out/prof_src python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_src.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_src.log
