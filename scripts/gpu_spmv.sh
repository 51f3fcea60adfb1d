set -x
timeout 600 python bench.py --workload spmv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_spmv.json 2> gpurun_out/bench_spmv.err; echo rc=$?
tail -3 gpurun_out/bench_spmv.err
