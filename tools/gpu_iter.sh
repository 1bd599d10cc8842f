cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "pipeline or taesd or dropin or cabi" > gpurun_out/t_pipe.txt 2>&1
echo "tests rc=$?" >> gpurun_out/t_pipe.txt
timeout 300 python bench.py --no-cpu-baseline --steps 40 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err
SDX_DECODE_OVERLAP=0 timeout 300 python bench.py --no-cpu-baseline --steps 40 --warmup 5 > gpurun_out/b1_noov.json 2>> gpurun_out/b1.err
timeout 300 python bench.py --no-cpu-baseline --steps 40 --warmup 5 --streams 8 --n-steps 1 --guidance self_negative > gpurun_out/b4.json 2>> gpurun_out/b1.err
SDX_DECODE_OVERLAP=0 timeout 300 python bench.py --no-cpu-baseline --steps 40 --warmup 5 --streams 8 --n-steps 1 --guidance self_negative > gpurun_out/b4_noov.json 2>> gpurun_out/b1.err
