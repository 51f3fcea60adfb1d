set -x
timeout 1200 python -m pytest tests -x -q -m gpu -k "spmv_full" -s > gpurun_out/q_spmvfull.log 2>&1; echo rc=$?
tail -5 gpurun_out/q_spmvfull.log
