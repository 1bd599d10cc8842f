"""Generates tests/golden/*.json from the reference compiled in this container
(oracle/_ref/libstagger_ref.so, built from /root/reference/proj/core/src by
oracle/Makefile).  The fixtures travel with the repo so GPU-box tests can pin
the oracle without /root/reference.  Run: python tests/golden/make_golden.py"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import load, make_cfg  # noqa: E402

ref = load("ref")
cases = []
for n in (1, 2, 4):
    for mode in ("none", "cfg", "self_negative", "onetime_negative"):
        for lcm in ("exact", "boundary_approx"):
            d = 16
            cfgd = dict(n_steps=n, guidance_mode=mode, d_latent=d, lcm_mode=lcm, seed=7)
            cfg = make_cfg(**cfgd)
            cond = ref.gaussian(ref.derive_seed(7, 4), d)
            neg = ref.gaussian(ref.derive_seed(7, 5), d) if mode in ("cfg", "onetime_negative") else None
            x0 = ref.gaussian(1234 + n, d)
            out = ref.sequential(cfg, cond, x0, neg)
            cases.append(dict(cfg=cfgd, cond=cond.tolist(), neg=None if neg is None else neg.tolist(),
                              x0=x0.tolist(), x0_hat=out.tolist()))
# SSF decisions over u8 frames (reference SsfState on integer-valued payloads)
rng = np.random.default_rng(5)
base = rng.integers(0, 256, 1024)
frames, dec = [], []
g = ref.ssf(0.98, ref.derive_seed(3, 2))
for i in range(300):
    f = base.copy()
    k = rng.integers(0, 200)
    idx = rng.integers(0, 1024, k)
    f[idx] = rng.integers(0, 256, k)
    if i % 50 == 49:
        base = rng.integers(0, 256, 1024)
    frames.append(f.astype(np.uint8).tolist())
    dec.append(g.gate(f.astype(np.float64)))
json.dump({"engine": cases, "ssf": {"eta": 0.98, "seed": int(ref.derive_seed(3, 2)), "frames": frames,
                                    "decisions": dec}},
          open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "engine_golden.json"), "w"))
print("wrote", len(cases), "engine cases,", len(dec), "ssf decisions")
