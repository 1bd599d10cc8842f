"""B200 analogues of the reference's bench tables (bench.cpp:225-285,
engine.cpp:240-309) with the real UNet + TAESD pipeline, measured by bench.py:

  stream_batch    n-step denoising as Stream Batch (one n-row UNet call per tick)
                  vs sequential (n one-row UNet calls per frame) vs wait-and-batch
                  (n calls of an n-frame batch: same work as Stream Batch, latency 2n)
  guidance        frames/s and UNet rows per frame for none / cfg / self-negative /
                  onetime-negative (R-CFG) at n = 1 and 4
  ssf             the similarity filter on a near-static vs a dynamic stream

Each entry is one `python bench.py ...` run (device-timed, resident frames);
sequential and wait-and-batch per-frame times are composed from the measured
stage times (denoiser at 1 and n rows, codec, control), as the reference does
from its cost model.

    python tools/bench_tables.py [--out gpurun_out/bench_tables]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(*args):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline", "--steps", "24", "--warmup", "4",
           *args]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    if p.returncode != 0:
        raise RuntimeError(p.stderr[-2000:])
    return json.loads(p.stdout.strip().splitlines()[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "bench_tables"))
    args = ap.parse_args()
    res = {"stream_batch": [], "guidance": [], "ssf": []}
    one = bench("--n-steps", "1")
    st1 = one["stage_ms_per_step"]
    den1 = st1["denoiser"]
    codec = st1["encode"] + st1["decode"]
    other = st1["ssf"] + st1["control"] + st1["step"]
    for n in (1, 2, 4):
        r = bench("--n-steps", str(n)) if n > 1 else one
        st = r["stage_ms_per_step"]
        stream_ms = r["ms_per_step"]  # one output frame per step at steady state
        seq_ms = n * den1 + codec + n * (other)
        wab_ms = st["denoiser"] + codec + other  # n calls of n rows for n frames == per frame one n-row call
        res["stream_batch"].append({"n": n, "sequential_ms": round(seq_ms, 3), "stream_ms": round(stream_ms, 3),
                                    "wait_and_batch_ms": round(wab_ms, 3), "speedup": round(seq_ms / stream_ms, 3),
                                    "stream_latency_ticks": n, "wait_and_batch_latency_ticks": 2 * n,
                                    "unet_ms_n_rows": round(st["denoiser"], 3), "unet_ms_1_row": round(den1, 3),
                                    "fps": r["value"]})
    rows_per_frame = {"none": lambda n: n, "cfg": lambda n: 2 * n, "self_negative": lambda n: n,
                      "onetime_negative": lambda n: n + 1}
    for n in (1, 4):
        row = {"n": n}
        for mode in ("none", "cfg", "self_negative", "onetime_negative"):
            r = bench("--n-steps", str(n), "--guidance", mode)
            row[f"{mode}_ms"] = r["ms_per_step"]
            row[f"{mode}_fps"] = r["value"]
            row[f"{mode}_unet_rows_per_frame"] = rows_per_frame[mode](n)
        row["cfg_over_self"] = round(row["cfg_ms"] / row["self_negative_ms"], 3)
        row["cfg_over_onetime"] = round(row["cfg_ms"] / row["onetime_negative_ms"], 3)
        res["guidance"].append(row)
    for label, extra in (("ssf on", []), ("ssf off", ["--no-ssf"])):
        r = bench("--n-steps", "4", *extra)
        res["ssf"].append({"config": label, "fps": r["value"], "ms_per_step": r["ms_per_step"],
                           "denoiser_ms": r["stage_ms_per_step"]["denoiser"]})
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out + ".json", "w"), indent=1)
    lines = ["# B200 bench tables (bench.py, 1 B200, UNet + TAESD 512x512, device-timed)", "",
             "## stream_batch (bench.cpp:225-244, engine.cpp:240-309)", "",
             "| n | sequential ms/frame | stream ms/frame | wait-and-batch ms/frame | speedup | latency stream / w&b (ticks) |",
             "|---|---|---|---|---|---|"]
    for r in res["stream_batch"]:
        lines.append(f"| {r['n']} | {r['sequential_ms']} | {r['stream_ms']} | {r['wait_and_batch_ms']} | {r['speedup']} | "
                     f"{r['stream_latency_ticks']} / {r['wait_and_batch_latency_ticks']} |")
    lines += ["", "## guidance (bench.cpp:246-280)", "",
              "| n | none ms | cfg ms | self-neg ms | onetime ms | cfg/self | cfg/onetime | UNet rows/frame (none, cfg, self, onetime) |",
              "|---|---|---|---|---|---|---|---|"]
    for r in res["guidance"]:
        lines.append(f"| {r['n']} | {r['none_ms']} | {r['cfg_ms']} | {r['self_negative_ms']} | {r['onetime_negative_ms']} | "
                     f"{r['cfg_over_self']} | {r['cfg_over_onetime']} | {r['none_unet_rows_per_frame']}, "
                     f"{r['cfg_unet_rows_per_frame']}, {r['self_negative_unet_rows_per_frame']}, "
                     f"{r['onetime_negative_unet_rows_per_frame']} |")
    lines += ["", "## ssf (bench stream: moving gradients + noise, eta 0.98)", "", "| config | frames/s | ms/step |",
              "|---|---|---|"]
    for r in res["ssf"]:
        lines.append(f"| {r['config']} | {r['fps']} | {r['ms_per_step']} |")
    open(args.out + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
