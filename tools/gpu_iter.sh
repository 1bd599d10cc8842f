cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_unet_gpu.py tests/test_pipeline_unet_gpu.py -x -q > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 600 python bench.py --streams 8 --n-steps 1 --guidance self_negative --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --no-cpu-baseline --no-graph --steps 10 > gpurun_out/bench_cfg1_nograph.json 2> gpurun_out/bench_cfg1_nograph.err
tail -2 gpurun_out/pytest_k.log
