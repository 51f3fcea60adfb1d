# SORT vs CUB on the library's own key sets, and the SORT / HASH / SEGMENT crossover (bench per dedup mode)
set -x
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/cub_sort scripts/cub_sort.cu
for w in sgemm stencil spmv; do
  python scripts/dump_keys.py $w /tmp/keys_$w.bin > gpurun_out/dump_$w.log 2>&1
  /tmp/cub_sort /tmp/keys_$w.bin > gpurun_out/cub_$w.json; cat gpurun_out/cub_$w.json; rm -f /tmp/keys_$w.bin
  for d in sort hash segment; do timeout 900 python bench.py --workload $w --only --dedup $d --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mode_${w}_$d.json 2> gpurun_out/mode_${w}_$d.err; echo rc=$?; done
done
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"thermo::onesweep_kernel" -s 2 -c 1 -o gpurun_out/r2_prof_onesweep_stencil python bench.py --workload stencil --only --dedup sort --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_onesweep.log 2>&1; echo rc=$?
python scripts/ncu_metrics.py gpurun_out/r2_prof_onesweep_stencil.ncu-rep > gpurun_out/r2_prof_onesweep_stencil.json
