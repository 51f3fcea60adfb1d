set -x
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"seg_|decode_kernel" -s 8 -c 6 -o gpurun_out/prof_seg python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_seg.log 2>&1; echo rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"thermo::" --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches.log 2>&1; echo rc=$?
