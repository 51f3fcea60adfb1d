set -x
for m in sort hash; do
timeout 300 python bench.py --workload stencil --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --dedup $m > gpurun_out/bench_st_$m.json 2> gpurun_out/bench_st_$m.err; echo rc=$?
tail -2 gpurun_out/bench_st_$m.err
done
