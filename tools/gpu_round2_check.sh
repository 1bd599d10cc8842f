cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.txt 2>&1; echo "rc=$?" >> gpurun_out/t_all.txt
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 900 python tools/bench_tables.py --out gpurun_out/bench_tables > gpurun_out/bench_tables.log 2>&1
tail -3 gpurun_out/t_all.txt; cat gpurun_out/b1.json; tail -30 gpurun_out/bench_tables.log
