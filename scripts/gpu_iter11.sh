# parity + benches: chunk-id scatter, vectorised hist; decoder-side counting for all sector spaces (A/B)
set -x
timeout 1200 python -m pytest tests -x -q -m gpu --timeout 600 > gpurun_out/par_full.log 2>&1; echo rc=$?
tail -3 gpurun_out/par_full.log
b() { timeout 900 python bench.py --workload $1 --steps $2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$1', '$THERMO_SEG_COUNT_ALL', d['ms_per_step'], d['phase_ms'])"; }
b sgemm 10
b stencil 3
b synthetic 3
b spmv 2
export THERMO_SEG_COUNT_ALL=1
b synthetic 3
b spmv 2
