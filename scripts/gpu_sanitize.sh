# compute-sanitizer passes over smoke() and small parity tests of every kernel family:
# memcheck, racecheck (shared-memory hazards), synccheck
set -x
K="small_workloads or random_traces and 1- or warp_records_random and 1- or hot_sector or access_counts and tiny or sampled_block or run_compression and 0 or many_objects or window or whitelist or dense_multi or both_decoders or random_hot_cv or one_hot or pc_count"
for tool in memcheck racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --error-exitcode 17 --print-limit 10000 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/san_smoke_$tool.log 2>&1; echo smoke-$tool rc=$?
grep "SUMMARY" gpurun_out/san_smoke_$tool.log
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 17 --print-limit 10000 python -m pytest tests -q -m gpu -k "$K" -p no:cacheprovider > gpurun_out/san_tests_$tool.log 2>&1; echo tests-$tool rc=$?
grep "SUMMARY\|passed\|failed" gpurun_out/san_tests_$tool.log | tail -3
done
