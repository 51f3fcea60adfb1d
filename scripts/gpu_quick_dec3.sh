set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "small_workloads or random_traces or many_objects or window or hot_sector or synthetic_medium or gemm_full or stencil_full or sampled_block or access_counts" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -2 gpurun_out/q_pytest.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_b$i.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/q_b$i.json')); print('RES', 'ms/step %.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['phase_ms'].items()})"; done
timeout 300 python bench.py --workload stencil --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/q_st.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/q_st.json')); print('RES stencil', 'ms/step %.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['phase_ms'].items()})"
