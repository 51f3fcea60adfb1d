set -x
for m in sort hash; do
timeout 600 python bench.py --workload spmv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --dedup $m > gpurun_out/bench_spmv_$m.json 2> gpurun_out/bench_spmv_$m.err; echo rc=$?
done
