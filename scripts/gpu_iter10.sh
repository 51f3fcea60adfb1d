# launch lists of the synthetic and spmv configs (SEGMENT) + quick benches
set -x
timeout 600 python bench.py --workload synthetic --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_synth.json 2>gpurun_out/bench_synth.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_synth.json'));print('synth', d['value'], d['ms_per_step'], d['phase_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"thermo::" --csv --log-file gpurun_out/launches_synth.csv python bench.py --workload synthetic --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_synth.log 2>&1; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"thermo::" --csv --log-file gpurun_out/launches_spmv.csv python bench.py --workload spmv --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_spmv.log 2>&1; echo rc=$?
