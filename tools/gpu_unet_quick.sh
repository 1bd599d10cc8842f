# GEMM/UNet parity tests + per-op profile at 4 rows + model-picked GEMM timings
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_unet_gpu.py -q -x > gpurun_out/t_kern.txt 2>&1; echo "rc=$?" >> gpurun_out/t_kern.txt
timeout 300 python tools/prof_ops.py 4 > gpurun_out/prof_ops_r4.txt 2>&1
SDX_SWEEP_MODEL_ONLY=1 timeout 300 python tools/gemm_sweep.py 4 > gpurun_out/gemm_quick.txt 2>&1
tail -2 gpurun_out/t_kern.txt; head -16 gpurun_out/prof_ops_r4.txt; tail -1 gpurun_out/gemm_quick.txt
