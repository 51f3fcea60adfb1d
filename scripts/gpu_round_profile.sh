# the round's evidence: default bench line, reference arm, warp-format line, ncu launch list, one full capture per hot kernel
set -x
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo rc=$?
timeout 600 python bench.py --format warp --no-cpu-baseline > gpurun_out/bench_warpfmt.json 2> gpurun_out/bench_warpfmt.err; echo rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"thermo::" --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches.log 2>&1; echo rc=$?
timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::(decode_kernel|seg_chunk|seg_scatter)" -s 3 -c 3 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo rc=$?
