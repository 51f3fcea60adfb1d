# decode with shared-memory window / pc caches: 3 vs 4 blocks per SM; parity of the decode-heavy tests
set -x
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -k "small or fuzz or random or warp or hot or block or gemm" > gpurun_out/par_q.log 2>&1; echo rc=$?
tail -2 gpurun_out/par_q.log
for m in 3 4 3 4; do THERMO_DEC_MINB=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>gpurun_out/b.err; python -c "import json;d=json.load(open('gpurun_out/b.json'));print($m, d['ms_per_step'], d['phase_ms']['ms_decode'])"; done
