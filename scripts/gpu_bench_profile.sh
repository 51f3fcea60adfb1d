set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_sort.json 2> gpurun_out/bench_sort.err; echo rc=$?
timeout 400 python bench.py --steps 5 --warmup 3 --dedup hash --no-cpu-baseline --no-e2e > gpurun_out/bench_hash.json 2> gpurun_out/bench_hash.err; echo rc=$?
KS='regex:decode|find_heads|onesweep|sort_|count_|object_hist|pc_hist|indicator|hash_'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KS" --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_list.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -o gpurun_out/prof_decode python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_decode.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"onesweep|count_sorted|sort_hist" -s 9 -c 4 -o gpurun_out/prof_sort python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sort.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests -x -q -m gpu -k full_size > gpurun_out/full.log 2>&1; echo rc=$?
