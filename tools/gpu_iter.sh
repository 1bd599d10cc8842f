cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k attention > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
timeout 600 python tools/attn_probe.py > gpurun_out/attn_probe.txt 2>&1
tail -2 gpurun_out/pytest_k.log
