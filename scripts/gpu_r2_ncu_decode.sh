# ncu --set full with source of the decode kernels on a workload (one launch each: the lane-per-record
# decoder on SpMV, the per-instruction view kernel elsewhere, and the general kernel)
set -x
W=${W:-spmv}
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::(decode_kernel|decode_lane_kernel|decode_general_kernel)" -c 2 -o gpurun_out/r2_prof_decode_$W python bench.py --workload $W --only --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_decode_$W.log 2>&1; echo rc=$?
python scripts/ncu_metrics.py gpurun_out/r2_prof_decode_$W.ncu-rep > gpurun_out/r2_prof_decode_$W.json
