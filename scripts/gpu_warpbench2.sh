set -x
timeout 300 python -m pytest tests -x -q -m gpu -k "warp_records" --timeout 120 > gpurun_out/par.log 2>&1; echo rc=$?
tail -2 gpurun_out/par.log
timeout 300 python bench.py --format warp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_warp.json 2> gpurun_out/bench_warp.err; echo rc=$?
