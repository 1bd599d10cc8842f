cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k groupnorm > gpurun_out/t_gn.txt 2>&1
timeout 300 python tools/gn_bench.py 4 > gpurun_out/gn_bench.txt 2>&1
timeout 300 python tools/gn_bench.py 8 >> gpurun_out/gn_bench.txt 2>&1
