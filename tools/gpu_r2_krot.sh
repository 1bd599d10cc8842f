cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_unet_gpu.py -q -x > gpurun_out/t_kern.txt 2>&1; echo "rc=$?" >> gpurun_out/t_kern.txt
tail -2 gpurun_out/t_kern.txt
echo "== krot on"; timeout 300 python tools/gemm_probe.py
echo "== krot off"; SDX_KROT=0 timeout 300 python tools/gemm_probe.py
bash tools/ab_env.sh "SDX_KROT=0" 4
bash tools/ab_env.sh "SDX_KROT=0" 8
