cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_unet_gpu.py tests/test_pipeline_unet_gpu.py -m gpu -x -q > gpurun_out/t_all.txt 2>&1
timeout 300 python tools/prof_ops.py 4 > gpurun_out/prof_ops_r4.txt 2>&1
timeout 300 python tools/prof_ops.py 8 > gpurun_out/prof_ops_r8.txt 2>&1
