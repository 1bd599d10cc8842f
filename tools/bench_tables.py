"""B200 analogues of the reference's bench tables (bench.cpp:225-285,
engine.cpp:213-309) with the real UNet + TAESD, all device-timed:

  stream_batch    n-step denoising three ways, each MEASURED as one CUDA graph:
                  Stream Batch (bench.py: the full pipeline, one n-row UNet call per
                  tick), sequential (per frame: encode, n one-row UNet calls, decode;
                  sdx_bench_denoise_loop(1, n, 1)) and wait-and-batch (per n frames:
                  encode n, n calls of n rows, decode n; sdx_bench_denoise_loop(n, n, n)).
                  The sequential / wait-and-batch graphs leave out the SSF gate and the
                  fused step kernel (~0.03 ms per frame, see the stage times).
  guidance        frames/s and UNet rows per frame for none / cfg / self-negative /
                  onetime-negative (R-CFG) at n = 1 and 4
  ssf             the similarity filter on a dynamic and a near-static scene, on and
                  off, with the measured skip rate

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


def denoise_loop(rows, calls, frames, n, iters=12):
    import ctypes as C

    sys.path.insert(0, ROOT)
    from paper_2312_12491_b200 import _lib as L

    f = L.lib.sdx_bench_denoise_loop
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.POINTER(C.c_double)]
    ms = C.c_double()
    st = f(rows, calls, frames, n, iters, 0, 0, C.byref(ms))
    if st != 0:
        raise RuntimeError(L.lib.sdx_last_error())
    return ms.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "bench_tables"))
    args = ap.parse_args()
    res = {"stream_batch": [], "guidance": [], "ssf": []}
    for n in (1, 2, 4):
        r = bench("--n-steps", str(n))
        stream_ms = r["ms_per_step"]  # one output frame per step at steady state
        seq_ms = denoise_loop(1, n, 1, n)
        wab_ms = denoise_loop(n, n, n, n) / n
        res["stream_batch"].append({"n": n, "sequential_ms": round(seq_ms, 3), "stream_ms": round(stream_ms, 3),
                                    "wait_and_batch_ms": round(wab_ms, 3), "speedup": round(seq_ms / stream_ms, 3),
                                    "stream_latency_ticks": n, "wait_and_batch_latency_ticks": 2 * n,
                                    "unet_ms_n_rows": r["stage_ms_per_step"]["denoiser"], "fps": r["value"]})
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
    for scene in ("dynamic", "near-static"):
        for label, extra in (("on", []), ("off", ["--no-ssf"])):
            r = bench("--n-steps", "4", "--scene", scene, *extra)
            res["ssf"].append({"scene": scene, "ssf": label, "fps": r["value"], "ms_per_step": r["ms_per_step"],
                               "skip_rate": r["config"]["ssf_skip_rate"],
                               "denoiser_ms": r["stage_ms_per_step"]["denoiser"]})
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out + ".json", "w"), indent=1)
    lines = ["# B200 bench tables (1 B200, UNet + TAESD 512x512, every column device-timed)", "",
             "## stream_batch (bench.cpp:225-244, engine.cpp:240-309)", "",
             "sequential and wait-and-batch: one CUDA graph of encode + UNet calls + decode "
             "(sdx_bench_denoise_loop); stream: the full pipeline (bench.py)", "",
             "| n | sequential ms/frame | stream ms/frame | wait-and-batch ms/frame | speedup vs sequential | latency stream / w&b (ticks) |",
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
    lines += ["", "## ssf (eta 0.98, 4-step; the near-static scene redraws ~2% of the bytes per frame)", "",
              "| scene | SSF | frames/s | ms/step | skip rate | UNet ms/step |", "|---|---|---|---|---|---|"]
    for r in res["ssf"]:
        lines.append(f"| {r['scene']} | {r['ssf']} | {r['fps']} | {r['ms_per_step']} | {r['skip_rate']} | "
                     f"{r['denoiser_ms']} |")
    open(args.out + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
