"""Summarise a bench.py JSON line from stdin: value, e2e, roofline frac, clocks, stage times."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
st = d.get("stage_ms_per_step", {})
print(f"{d['value']:.2f} fps e2e {d['e2e']['value']:.2f} frac {d['roofline']['frac']:.3f} clk {d['clocks']['sm_mhz']}"
      f" den {st.get('denoiser', 0):.3f} enc {st.get('encode', 0):.3f} dec {st.get('decode', 0):.3f}")
