cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 600 python bench.py --streams 8 --n-steps 1 --guidance self_negative --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
