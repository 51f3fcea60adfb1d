# ncu --set full with source of the lane decoder on SpMV (one launch)
set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::decode_lane_kernel" -s 1 -c 1 -o gpurun_out/r2_prof_lane_spmv python bench.py --workload spmv --only --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_lane.log 2>&1; echo rc=$?
python scripts/ncu_metrics.py gpurun_out/r2_prof_lane_spmv.ncu-rep > gpurun_out/r2_prof_lane_spmv.json
