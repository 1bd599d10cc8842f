# GEMM kernel tests + probes + model-picked UNet shapes + whole-forward time
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_unet_gpu.py -q -x > gpurun_out/t_kern.txt 2>&1; echo "rc=$?" >> gpurun_out/t_kern.txt
timeout 300 python tools/gemm_probe.py > gpurun_out/probe.txt 2>&1
SDX_SWEEP_MODEL_ONLY=1 timeout 300 python tools/gemm_sweep.py 4 > gpurun_out/gemm_quick.txt 2>&1
timeout 200 python tools/unet_time.py 4 8 > gpurun_out/ut.txt 2>&1
tail -2 gpurun_out/t_kern.txt; cat gpurun_out/probe.txt; tail -1 gpurun_out/gemm_quick.txt; cat gpurun_out/ut.txt
