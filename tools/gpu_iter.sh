cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "attention or tilings or conv3x3_halo" > gpurun_out/memcheck_kernels.txt 2>&1
echo "rc=$?" >> gpurun_out/memcheck_kernels.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_unet_gpu.py -m gpu -x -q > gpurun_out/memcheck_unet.txt 2>&1
echo "rc=$?" >> gpurun_out/memcheck_unet.txt
