cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k attention > gpurun_out/t_attn.txt 2>&1
timeout 300 python tools/attn_probe.py > gpurun_out/attn_probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.txt 2>&1
timeout 300 python tools/prof_ops.py 4 > gpurun_out/prof_ops_r4.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 40 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 300 python bench.py --no-cpu-baseline --steps 40 --warmup 5 --streams 8 --n-steps 1 --guidance self_negative > gpurun_out/b4.json 2>> gpurun_out/b1.err
