# ncu --set full of the count-phase kernels on the given workload (one launch each)
set -x
W=${W:-spmv}
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::(seg_coarse_kernel|seg_fine_kernel|seg_chunk_kernel|seg_big_kernel|seg_big_pc_kernel)" -c 5 -o gpurun_out/r2_prof_count_$W python bench.py --workload $W --only --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_count_$W.log 2>&1; echo rc=$?
python scripts/ncu_metrics.py gpurun_out/r2_prof_count_$W.ncu-rep > gpurun_out/r2_prof_count_$W.json; echo rc=$?
