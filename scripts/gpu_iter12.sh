# decode occupancy/register trade-off: 2 blocks (102 regs) vs 3 blocks (78 regs)
set -x
for m in 3 2 3 2; do THERMO_DEC_MINB=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>gpurun_out/b.err; python -c "import json;d=json.load(open('gpurun_out/b.json'));print($m, d['ms_per_step'], d['phase_ms']['ms_decode'])"; done
