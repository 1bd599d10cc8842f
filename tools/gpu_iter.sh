cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2400 python tools/bench_tables.py --out gpurun_out/bench_tables > gpurun_out/bench_tables.log 2>&1
