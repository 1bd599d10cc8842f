cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" 2>&1 | tail -1
timeout 300 python tools/attn_time.py
timeout 300 python tools/attn_timeline.py 4 4096 5 | tail -10
