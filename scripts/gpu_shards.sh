set -x
timeout 600 python -m pytest tests/test_gpu_shards.py -x -q --timeout 120 > gpurun_out/shards.log 2>&1; echo rc=$?
tail -30 gpurun_out/shards.log
