# launch lists (one step) of the irregular workloads: where the count phase goes
set -x
for w in stencil spmv synthetic; do
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k regex:"thermo::" --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_$w.log 2>&1; echo rc=$?
done
