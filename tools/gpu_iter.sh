cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python tools/gemm_sweep.py 4 8 > gpurun_out/gemm_sweep.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
