# final tree check: the whole GPU suite, smoke, one default bench line
set -x
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/final_pytest.log 2>&1; echo rc=$?
tail -3 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo rc=$?
tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo rc=$?
cat gpurun_out/final_bench.json | head -c 600
