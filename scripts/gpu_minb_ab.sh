# decode occupancy A/B: THERMO_DEC_MINB=3 (default) vs 4 (64 registers, 4 blocks/SM when the smem fits)
set -x
THERMO_DEC_MINB=4 timeout 600 python -m pytest tests -x -q -m gpu -k "small_workloads or random_traces or many_objects or window or hot_sector or synthetic_medium" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -2 gpurun_out/q_pytest.log
for v in 3 4 3 4; do THERMO_DEC_MINB=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/q_minb_$v.json 2> gpurun_out/q_minb_$v.err; echo rc=$?;
python -c "
import json; d=json.load(open('gpurun_out/q_minb_$v.json')); print('minb $v', 'ms/step %.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['phase_ms'].items()})"; done
THERMO_DEC_MINB=4 timeout 300 python bench.py --workload stencil --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/q_minb_st4.json 2>&1; echo rc=$?
THERMO_DEC_MINB=3 timeout 300 python bench.py --workload stencil --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/q_minb_st3.json 2>&1; echo rc=$?
for v in st3 st4; do python -c "
import json; d=json.load(open('gpurun_out/q_minb_$v.json')); print('minb $v', 'ms/step %.3f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['phase_ms'].items()})"; done
timeout 400 env THERMO_DEC_MINB=4 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"thermo::decode_kernel" -s 3 -c 1 -o gpurun_out/prof_dec4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_dec4.log 2>&1; echo rc=$?
