# ncu launch lists (time + DRAM bytes per kernel) of the given workloads
set -x
for w in ${WL:-stencil spmv}; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k regex:"thermo::" --csv --log-file gpurun_out/ll_$w.csv python bench.py --workload $w --only --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ll_$w.log 2>&1; echo rc=$?
python scripts/launch_table.py gpurun_out/ll_$w.csv
done
