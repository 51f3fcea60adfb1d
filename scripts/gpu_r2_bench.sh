# the default bench line (headline SpMV + other configs); LAUNCH=1: first the launch lists of every config + traffic table
set -x
if [ "${LAUNCH:-0}" = "1" ]; then
WL="sgemm stencil spmv synthetic" bash scripts/gpu_r2_launch.sh
python scripts/traffic_from_launches.py sgemm=gpurun_out/ll_sgemm.csv stencil=gpurun_out/ll_stencil.csv spmv=gpurun_out/ll_spmv.csv synthetic=gpurun_out/ll_synthetic.csv > profiles/r2_traffic.json
cp profiles/r2_traffic.json gpurun_out/r2_traffic.json
fi
s=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$? elapsed=$(( $(date +%s) - s ))
tail -20 gpurun_out/bench_default.err
