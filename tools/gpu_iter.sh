cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_unet_gpu.py -x -q > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
timeout 300 python tools/prof_ops.py 4 1 > gpurun_out/prof_ops_r4.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
tail -2 gpurun_out/pytest_k.log
