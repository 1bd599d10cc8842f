cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/t_attn.txt 2>&1; echo "rc=$?" >> gpurun_out/t_attn.txt
: > gpurun_out/attn_time.txt
for v in 1 0 1; do echo "ts3=$v" >> gpurun_out/attn_time.txt; SDX_ATTN_TS3=$v timeout 300 python tools/attn_time.py >> gpurun_out/attn_time.txt 2>&1; done
grep -E "passed|failed|rc=" gpurun_out/t_attn.txt; cat gpurun_out/attn_time.txt
