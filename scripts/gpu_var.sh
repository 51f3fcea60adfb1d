timeout 300 python -m pytest tests -x -q -m gpu -k "not full_size" --timeout 120 > gpurun_out/par.log 2>&1; echo rc=$?
for i in 1 2 3; do
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_v$i.json 2> /dev/null
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,temperature.gpu,power.draw --format=csv > gpurun_out/smi.txt
