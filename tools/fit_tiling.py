"""Fit the constants of the tiling cost model (gemm_sm100.cu: gemm_cost) to a
recorded sweep (SDX_SWEEP_JSON=... python tools/gemm_sweep.py 2 4 8): the
objective is the summed measured time of the candidate the model would pick
per shape (restricted to the measured candidates).

    python tools/fit_tiling.py gpurun_out/sweep_all.json
"""
import json
import random
import sys
from collections import defaultdict

SM = 148


def cost(P, M, N, K, bn, s, res, out_bytes=2):
    pair = bn < 0
    bn = abs(bn)
    mu = 256 if pair else 128
    slots = SM // 2 if pair else SM
    mt, nt = -(-M // mu), -(-N // bn)
    units = mt * nt * s
    nk = K // 64
    bnl = bn / 2 if pair else bn
    nku = -(-nk // s)
    slice_ = max(P["a0"], P["a1"] * bn, P["a2"] * (128 + bnl)) + P["a3"]
    ml = nku * slice_
    eb = 4.0 if s > 1 else out_bytes + (2.0 if res else 0.0)
    epi = P["e0"] * 128.0 * bn * eb / 16.0 + P["e1"]
    per_cta = -(-units // slots)
    t = per_cta * max(ml, epi) + P["c0"] + min(ml, epi)
    if pair:
        t += P["p0"]
    if s > 1:
        t += P["s0"] + M * N * (4.0 * s + out_bytes + (2.0 if res else 0.0)) / (SM * P["s1"])
    return t


def main():
    recs = json.load(open(sys.argv[1]))
    shapes = defaultdict(dict)
    for r in recs:
        if r["N"] <= 64:
            continue  # TAESD 64-channel convs (halo-tiled, not planned by the model)
        if r["bn"] < 0 and (r["K"] < 11520 or -r["bn"] < 128):
            continue  # the planner's pair rule (choose_tiling)
        key = (r["label"], r["M"], r["N"], r["K"], r["res"])
        shapes[key][(r["bn"], r["s"])] = r["us"]
    best_total = sum(min(c.values()) for c in shapes.values())

    def objective(P):
        tot = 0.0
        for (lab, M, N, K, res), c in shapes.items():
            pick = min(c, key=lambda bs: cost(P, M, N, K, bs[0], bs[1], res))
            tot += c[pick]
        return tot

    P0 = {"a0": 0.0, "a1": 2.0, "a2": 2.0, "a3": 40.0, "e0": 1.0, "e1": 400.0, "c0": 1500.0, "p0": 0.0, "s0": 5000.0,
          "s1": 16.0}
    cur, cv = dict(P0), objective(P0)
    print(f"best possible {best_total:.1f} us, current model {cv:.1f} us over {len(shapes)} shapes")
    random.seed(1)
    scales = {"a0": 200.0, "a1": 0.5, "a2": 0.5, "a3": 50.0, "e0": 0.3, "e1": 300.0, "c0": 1000.0, "p0": 1000.0,
              "s0": 2000.0, "s1": 6.0}
    for it in range(6000):
        k = random.choice(list(scales))
        cand = dict(cur)
        cand[k] = max(0.0, cand[k] + random.gauss(0, scales[k]) * (1.0 if it < 4000 else 0.3))
        v = objective(cand)
        if v <= cv:
            cur, cv = cand, v
    print(f"fitted model {cv:.1f} us: " + ", ".join(f"{k}={v:.3g}" for k, v in cur.items()))
    for (lab, M, N, K, res), c in sorted(shapes.items()):
        pick = min(c, key=lambda bs: cost(cur, M, N, K, bs[0], bs[1], res))
        b = min(c, key=c.get)
        if c[pick] > 1.03 * c[b]:
            print(f"  {lab:44s} pick {pick} {c[pick]:.1f} us, best {b} {c[b]:.1f} us")


if __name__ == "__main__":
    main()
