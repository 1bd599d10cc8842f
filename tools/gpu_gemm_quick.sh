# model-picked tilings of every UNet GEMM / conv shape at 4 rows, graph-timed; GEMM parity tests
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x > gpurun_out/t_kern.txt 2>&1; echo "rc=$?" >> gpurun_out/t_kern.txt
SDX_SWEEP_MODEL_ONLY=1 timeout 300 python tools/gemm_sweep.py 4 > gpurun_out/gemm_quick.txt 2>&1
tail -2 gpurun_out/t_kern.txt; grep -v "^conv3x3 1x" gpurun_out/gemm_quick.txt | cut -c1-100
