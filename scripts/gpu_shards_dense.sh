set -x
timeout 600 python -m pytest tests/test_gpu_shards.py -x -q -k "dense_block or match_one_context and 0-" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -20 gpurun_out/q_pytest.log
