# round 2, first pass: the whole GPU suite on the current tree + per-config bench lines with stats
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r2_pytest_gpu.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_pytest_gpu.log
for w in spmv stencil; do timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err; echo rc=$?; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k regex:"thermo::" --csv --log-file gpurun_out/r2_launches_spmv.csv python bench.py --workload spmv --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_launches_spmv.log 2>&1; echo rc=$?
