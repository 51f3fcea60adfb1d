# quick iteration + ncu full captures of the count kernels on the stencil and the general decoder on SpMV
bash scripts/gpu_quick_iter.sh
set -x
timeout 300 python bench.py --workload spmv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_spmv.json 2> gpurun_out/q_spmv.err; echo rc=$?
timeout 500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::(seg_chunk_kernel|seg_scatter)" -s 6 -c 2 -o gpurun_out/prof_stencil python bench.py --workload stencil --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_stencil.log 2>&1; echo rc=$?
timeout 500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::decode_general" -s 3 -c 1 -o gpurun_out/prof_spmv python bench.py --workload spmv --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_spmv.log 2>&1; echo rc=$?
