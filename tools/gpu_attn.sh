cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/t_attn.txt 2>&1; echo "rc=$?" >> gpurun_out/t_attn.txt
SDX_ATTN_POLY=0 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" >> gpurun_out/t_attn.txt 2>&1; echo "rc=$?" >> gpurun_out/t_attn.txt
: > gpurun_out/attn_time.txt
for p in 0 6 4 3 2; do echo "poly=$p" >> gpurun_out/attn_time.txt; SDX_ATTN_POLY=$p timeout 300 python tools/attn_time.py >> gpurun_out/attn_time.txt 2>&1; done
timeout 300 python tools/attn_timeline.py 4 4096 5 > gpurun_out/attn_timeline.txt 2>&1
cat gpurun_out/t_attn.txt | grep -E "passed|failed|rc="; cat gpurun_out/attn_time.txt; head -8 gpurun_out/attn_timeline.txt; tail -2 gpurun_out/attn_timeline.txt
