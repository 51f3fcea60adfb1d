set -x
for m in segment sort hash; do
timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --dedup $m > gpurun_out/bench_$m.json 2> gpurun_out/bench_$m.err; echo rc=$?
done
