# round-2 evidence on the committed tree: GPU tests, smoke, launch lists + traffic, default bench line,
# reference arm, warp-format line, ncu --set full of the headline's dominant kernels, local shards
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 2400 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/ev_pytest_gpu.log 2>&1; echo rc=$?
tail -20 gpurun_out/ev_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ev_smoke.log 2>&1; echo rc=$?
LAUNCH=1 bash scripts/gpu_r2_bench.sh
cp gpurun_out/bench_default.json gpurun_out/ev_bench_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev_bench_reference.json 2> gpurun_out/ev_bench_reference.err; echo rc=$?
timeout 900 python bench.py --workload sgemm --only --format warp --no-cpu-baseline > gpurun_out/ev_bench_warp.json 2> gpurun_out/ev_bench_warp.err; echo rc=$?
W=spmv bash scripts/gpu_r2_ncu_decode.sh
W=spmv bash scripts/gpu_r2_ncu_count.sh
W=sgemm bash scripts/gpu_r2_ncu_view.sh
for P in 1 2 4 8; do timeout 900 python bench.py --workload synthetic --local-shards $P --steps 2 --warmup 1 > gpurun_out/ev_shards_P$P.json 2> gpurun_out/ev_shards_P$P.err; echo rc=$?; done
