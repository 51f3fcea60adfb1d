set -x
timeout 600 python bench.py --workload spmv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --dedup hash > gpurun_out/bench_spmv_hash.json 2> gpurun_out/e1.err; echo rc=$?
timeout 600 python bench.py --workload stencil --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --dedup hash > gpurun_out/bench_st_hash.json 2> gpurun_out/e2.err; echo rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --dedup hash > gpurun_out/bench_sg_hash.json 2> gpurun_out/e3.err; echo rc=$?
