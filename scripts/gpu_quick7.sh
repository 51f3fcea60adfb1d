set -x
timeout 300 python -m pytest tests -x -q -m gpu -k "not full_size" --timeout 120 > gpurun_out/par.log 2>&1; echo rc=$?
tail -3 gpurun_out/par.log
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo rc=$?
timeout 200 python bench.py --workload stencil --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_st.json 2>gpurun_out/bench_st.err; echo rc=$?
timeout 600 python bench.py --workload spmv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --dedup segment > gpurun_out/bench_spmv.json 2> gpurun_out/bench_spmv.err; echo rc=$?
