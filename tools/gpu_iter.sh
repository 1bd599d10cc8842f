cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python tools/gemm_probe.py bn > gpurun_out/gemm_probe_bn.txt 2>&1
