set -x
timeout 300 python bench.py --format warp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_warp.json 2> gpurun_out/bench_warp.err; echo rc=$?
tail -3 gpurun_out/bench_warp.err
timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::decode_warp" -s 2 -c 1 -o gpurun_out/prof_warp python bench.py --format warp --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_w.log 2>&1; echo rc=$?
