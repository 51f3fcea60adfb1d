# SEGMENT iteration: parity of every SEGMENT case (small, fuzz, hot sectors, many objects, windows, full sizes) + bench lines
set -x
timeout 1500 python -m pytest tests -x -q -m gpu -k "small_workloads or random_traces or hot_sector or many_objects or window or synthetic_medium or full_size or shards or spmv_full" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -3 gpurun_out/q_pytest.log
for w in sgemm stencil spmv synthetic; do timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err; python -c "
import json; d=json.load(open('gpurun_out/q_$w.json')); print('RES $w', 'ms/step %.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['phase_ms'].items()})"; done
