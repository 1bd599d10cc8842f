cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
timeout 2400 python tools/bench_tables.py --out gpurun_out/bench_tables > gpurun_out/bench_tables.log 2>&1
