cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for lf in 0 1; do
SDX_LN_FOLD=$lf timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_ln${lf}.json 2>/dev/null
SDX_LN_FOLD=$lf timeout 600 python bench.py --streams 8 --n-steps 1 --guidance self_negative --no-cpu-baseline --steps 30 > gpurun_out/bench4_ln${lf}.json 2>/dev/null
done
SDX_LN_FOLD=1 timeout 600 python -m pytest tests/test_unet_gpu.py -x -q > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
tail -2 gpurun_out/pytest_k.log
