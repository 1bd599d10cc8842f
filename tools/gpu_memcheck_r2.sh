# compute-sanitizer memcheck / racecheck of the round-2 kernels (TAESD head/tail on mma.sync,
# GEMM producer / weight prefetch, GroupNorm DSMEM reads)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
CS="compute-sanitizer --tool memcheck --error-exitcode 9"
timeout 900 $CS python -m pytest tests/test_taesd_gpu.py -q -x > gpurun_out/memcheck_taesd.txt 2>&1; echo "rc=$?" >> gpurun_out/memcheck_taesd.txt
timeout 900 $CS python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm or conv or groupnorm" > gpurun_out/memcheck_kernels.txt 2>&1; echo "rc=$?" >> gpurun_out/memcheck_kernels.txt
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_taesd_gpu.py -q -x -k decoder > gpurun_out/racecheck_taesd.txt 2>&1; echo "rc=$?" >> gpurun_out/racecheck_taesd.txt
for f in gpurun_out/memcheck_taesd.txt gpurun_out/memcheck_kernels.txt gpurun_out/racecheck_taesd.txt; do tail -n 4 $f; done #/memcheck_taesd.txt gpurun_out/memcheck_kernels.txt gpurun_out/racecheck_taesd.txt
