# ncu --set full with source of the per-instruction view decoder on a workload (one launch)
set -x
W=${W:-stencil}
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::decode_kernel" -c 1 -o gpurun_out/r2_prof_view_$W python bench.py --workload $W --only --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_view_$W.log 2>&1; echo rc=$?
python scripts/ncu_metrics.py gpurun_out/r2_prof_view_$W.ncu-rep > gpurun_out/r2_prof_view_$W.json
