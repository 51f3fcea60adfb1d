# decode occupancy sweep: THERMO_DEC_MINB = 3 (default), 2, 4
set -x
for v in 3 2 4 3; do THERMO_DEC_MINB=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/mb_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/mb_$v.json')); print('RES $v', 'ms/step %.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['phase_ms'].items()})"; done
