# sharded mode: GPU tests + per-rank storage / work of P = 1, 2, 4, 8 in-process shards on the synthetic slice
set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "shards or smoke" > gpurun_out/shards_pytest.log 2>&1; echo rc=$?
tail -3 gpurun_out/shards_pytest.log
for P in 1 2 4 8; do timeout 900 python bench.py --workload synthetic --local-shards $P --steps 2 --warmup 1 > gpurun_out/shards_P$P.json 2> gpurun_out/shards_P$P.err; echo rc=$?; tail -3 gpurun_out/shards_P$P.err; done
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo rc=$?; tail -2 gpurun_out/smoke.log
