# full ncu captures of the sweep/scatter kernels on the synthetic config
set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::(seg_scatter_kernel|seg_chunk_kernel|object_hist_kernel|indicator_tile_kernel|seg_hist_kernel)" -s 5 -c 5 -o gpurun_out/prof_synth python bench.py --workload synthetic --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_synth.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_synth.log
