cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_pipeline_gpu.py tests/test_pipeline_unet_gpu.py -m gpu -x -q > gpurun_out/memcheck_pipeline.txt 2>&1
echo "rc=$?" >> gpurun_out/memcheck_pipeline.txt
