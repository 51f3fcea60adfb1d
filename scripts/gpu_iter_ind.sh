# indicator iteration: parity of every classify output (small, fuzz, synthetic medium, shards) + bench lines
set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "small_workloads or random_traces or synthetic_medium or many_objects or shards" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -2 gpurun_out/q_pytest.log
for w in sgemm synthetic spmv stencil; do timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err; python -c "
import json; d=json.load(open('gpurun_out/q_$w.json')); print('$w', 'ms/step %.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['phase_ms'].items()})"; done
