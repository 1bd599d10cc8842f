# headline (cfg1) and cfg4 bench lines, no CPU baseline
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 300 python bench.py --streams 8 --n-steps 1 --guidance self_negative --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b4.json 2> gpurun_out/b4.err
python - <<'PY'
import json
for f in ("gpurun_out/b1.json", "gpurun_out/b4.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], "fps e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], "clk", d["clocks"]["sm_mhz"], "stages", d["stage_ms_per_step"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-2000:])
PY
