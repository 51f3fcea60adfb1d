# full evidence pass on the current tree: GPU tests, smoke, bench lines (all workloads), launch list, ncu full of the hot kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo rc=$?
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo rc=$?
timeout 600 python bench.py --format warp --no-cpu-baseline > gpurun_out/bench_warpfmt.json 2> gpurun_out/bench_warpfmt.err; echo rc=$?
for w in stencil spmv synthetic; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo rc=$?; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"thermo::" --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches.log 2>&1; echo rc=$?
timeout 500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::(decode_kernel|seg_chunk_kernel|seg_scatter)" -s 3 -c 3 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo rc=$?
