# DENSE dedup (sampled-block mode): parity + timing against SEGMENT on the full SGEMM trace
set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "sampled_block or dense_multi or small_workloads or random_traces" > gpurun_out/q_pytest.log 2>&1; echo rc=$?
tail -3 gpurun_out/q_pytest.log
timeout 300 python scripts/dense_timing.py > gpurun_out/dense_timing.json 2> gpurun_out/dense_timing.err; echo rc=$?
cat gpurun_out/dense_timing.json; tail -3 gpurun_out/dense_timing.err
