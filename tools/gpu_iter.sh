cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.txt 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 60 --warmup 5 > gpurun_out/b1_p$i.json 2> gpurun_out/b1.err
SDX_STREAM_PRIO=0 timeout 300 python bench.py --no-cpu-baseline --steps 60 --warmup 5 > gpurun_out/b1_np$i.json 2>> gpurun_out/b1.err
timeout 300 python bench.py --no-cpu-baseline --steps 60 --warmup 5 --streams 8 --n-steps 1 --guidance self_negative > gpurun_out/b4_p$i.json 2>> gpurun_out/b1.err
SDX_STREAM_PRIO=0 timeout 300 python bench.py --no-cpu-baseline --steps 60 --warmup 5 --streams 8 --n-steps 1 --guidance self_negative > gpurun_out/b4_np$i.json 2>> gpurun_out/b1.err
done
