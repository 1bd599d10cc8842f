cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 600 python bench.py --streams 8 --n-steps 1 --guidance self_negative --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
SDX_GN_FUSE=1 SDX_LN_FOLD=1 timeout 600 python bench.py --streams 8 --n-steps 1 --guidance self_negative --no-cpu-baseline > gpurun_out/bench_cfg4_fused.json 2>/dev/null
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
