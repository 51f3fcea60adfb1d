set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "whitelist or sampled_block or dense_multi or warp_records or small_workloads" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -15 gpurun_out/q_pytest.log
