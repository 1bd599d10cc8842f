# Session start: full GPU tests, headline + cfg4 bench, whole-forward timer, per-op profile
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.txt 2>&1; echo "rc=$?" >> gpurun_out/t_all.txt
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 300 python bench.py --streams 8 --n-steps 1 --guidance self_negative --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b4.json 2> gpurun_out/b4.err
timeout 200 python tools/unet_time.py 4 8 > gpurun_out/unet_time.txt 2>&1
timeout 300 python tools/prof_ops.py 4 > gpurun_out/prof_ops_r4.txt 2>&1
tail -2 gpurun_out/t_all.txt
cat gpurun_out/unet_time.txt
python - <<'PY'
import json
for f in ("gpurun_out/b1.json", "gpurun_out/b4.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], "fps e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], "stages", d["stage_ms_per_step"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-2000:])
PY
head -20 gpurun_out/prof_ops_r4.txt
