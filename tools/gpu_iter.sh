cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.txt 2>&1
echo "tests rc=$?" >> gpurun_out/t_all.txt
timeout 300 python bench.py --no-cpu-baseline --steps 40 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 300 python bench.py --no-cpu-baseline --steps 40 --warmup 5 --streams 8 --n-steps 1 --guidance self_negative > gpurun_out/b4.json 2>> gpurun_out/b1.err
SDX_SWEEP_JSON=gpurun_out/sweep_fit.json timeout 2400 python tools/gemm_sweep.py 2 4 8 > gpurun_out/gemm_sweep_fit.txt 2>&1
