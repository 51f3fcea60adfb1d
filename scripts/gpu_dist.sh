set -x
timeout 600 python -m pytest tests/test_gpu_shards.py -x -q --timeout 120 > gpurun_out/shards.log 2>&1; echo rc=$?
tail -5 gpurun_out/shards.log
timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --force-dist > gpurun_out/bench_fd.json 2> gpurun_out/bench_fd.err; echo rc=$?
tail -3 gpurun_out/bench_fd.err
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tr1.json 2> gpurun_out/bench_tr1.err; echo rc=$?
tail -3 gpurun_out/bench_tr1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rc=$?
