# default bench line twice (clock sampling check) + one stencil line
set -x
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/qb_$i.json 2> gpurun_out/qb_$i.err; echo rc=$?; python -c "
import json; d=json.load(open('gpurun_out/qb_$i.json')); print('sgemm', 'ms/step %.3f' % d['ms_per_step'], d['clocks'], 'e2e %.3g' % d['e2e']['value'])"; done
timeout 300 python bench.py --workload stencil --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/qb_st.json 2> gpurun_out/qb_st.err; python -c "
import json; d=json.load(open('gpurun_out/qb_st.json')); print('stencil', 'ms/step %.3f' % d['ms_per_step'], d['clocks'])"
