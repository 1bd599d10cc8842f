#!/usr/bin/env python3
"""Benchmark of the B200 streaming denoise loop (contract: see DESIGN.md §Measurement).

One step = one pipeline iteration over every stream on every GPU: each stream
pushes one 3x512x512 u8 frame through the device SSF gate, encode, one batched
stream-batch tick (n in-flight frames per stream) and decode.  `value` is
output frames/s with the input frames already resident in HBM; `e2e` is the
same through the public C-ABI call (sdx_pipeline_push) from pinned host
frames, with the H2D of the frames and the D2H of the outputs inside the timed
region.  Multi-GPU: one process per GPU (torchrun), independent streams per
GPU, no collective on the data path; time = max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, W, C = 512, 512, 3
FRAME_BYTES = H * W * C


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--streams", type=int, default=8, help="independent streams per GPU")
    p.add_argument("--n-steps", type=int, default=4, help="denoising steps (in-flight frames per stream)")
    p.add_argument("--guidance", default="self_negative")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing (torch.distributed only for barrier / max-over-ranks)
# ---------------------------------------------------------------------------

class Dist:
    def __init__(self, backend):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist

            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        import torch

        dev = "cuda" if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class Clocks:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def synthetic_frames(rng, n_iter, S):
    """Dynamic 512x512 RGB scenes: moving gradient + noise, cosine to the
    previous frame well below eta, so every frame is processed (the gate still
    runs its full reduction)."""
    yy, xx = np.mgrid[0:H, 0:W]
    out = np.empty((n_iter, S, FRAME_BYTES), dtype=np.uint8)
    for i in range(n_iter):
        for s in range(S):
            img = np.stack([(xx * (1 + s) + 13 * i) % 256, (yy * (2 + s) + 7 * i) % 256,
                            rng.integers(0, 256, (H, W))], -1)
            out[i, s] = img.astype(np.uint8).reshape(-1)
    return out


def workload_cfg(args):
    from paper_2312_12491_b200 import stagger as sg

    d = FRAME_BYTES  # identity codec: latent = frame (TAESD codec not built yet)
    neg = None
    if args.guidance in ("cfg", "onetime_negative"):
        neg = sg.sample_gaussian(sg.derive_seed(0, 5), d)
    return sg.EngineConfig(n_steps=args.n_steps, guidance_mode=args.guidance, gamma=1.4, delta=1.0,
                           ssf_enabled=True, eta=0.98, seed=0, d_latent=d, negative_condition=neg)


def step_bytes_per_launch(n, guidance, d, S):
    """Algorithmic HBM bytes of one fused step launch at steady state (fp32):
    per in-flight row: read x (the entering row reads x0 + eps0 instead), the
    condition mean, eps_cached[next] (not on the terminal row), the reference
    latent (self: x0 / onetime: x0_ref, cfg: negative mean) and write the result."""
    per_stream = 0
    for step in range(n):
        b = 4 + 4  # mean + write
        b += 8 if step == 0 else 4
        if step < n - 1:
            b += 4
        if guidance in ("self_negative", "onetime_negative", "cfg"):
            b += 4
        if guidance == "onetime_negative" and step == 0:
            b += 4  # x0_ref write
        per_stream += b
    return per_stream * d * S


def run_ours(args, dist: Dist):
    import ctypes as C

    from paper_2312_12491_b200 import _lib as L
    from paper_2312_12491_b200 import stagger as sg

    dev = dist.local
    S = args.streams
    cfg = workload_cfg(args)
    ring = 4
    rng = np.random.default_rng(1000 + dist.rank)
    frames = synthetic_frames(rng, ring, S)
    p = sg.Pipeline(cfg, S, FRAME_BYTES, ring_depth=ring, device=dev)

    # ---- value: inputs resident in HBM ----
    p.upload_resident(frames)
    for _ in range(args.warmup):
        p.push_resident(copy_outputs=False)
    p.sync()
    p.set_profile(True)
    dist.barrier()
    with Clocks(dev) as clk:
        p.sync()
        p.reset_timer()
        for _ in range(args.steps):
            p.push_resident(copy_outputs=False)
        ms = p.device_time_ms()
        p.sync()
    kt = p.kernel_times()
    ms_max = dist.max(ms)
    frames_out = args.steps * S  # steady state: every stream emits one frame per iteration

    # ---- e2e: public API from pinned host frames, outputs copied back ----
    hp = C.c_void_p()
    nbytes = frames.nbytes
    assert L.lib.sdx_host_alloc(nbytes, C.byref(hp)) == 0
    host = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(hp.value)).reshape(frames.shape)
    host[:] = frames
    q = sg.Pipeline(cfg, S, FRAME_BYTES, ring_depth=ring, device=dev)
    got = 0
    for i in range(args.warmup):
        q.push_ptr(hp.value + (i % ring) * S * FRAME_BYTES)
        for s in range(S):
            q.pop_all(s)
    q.sync()
    dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        q.push_ptr(hp.value + (i % ring) * S * FRAME_BYTES)
        for s in range(S):
            got += len(q.pop_all(s))
    q.sync()
    for s in range(S):
        got += len(q.pop_all(s))
    e2e_s = time.perf_counter() - t0
    e2e_max = dist.max(e2e_s)
    q.close()
    L.lib.sdx_host_free(hp)

    step_ms = kt["step_ms"] / max(1, kt["step_launches"])
    ssf_ms = kt["ssf_ms"] / max(1, kt["ssf_launches"])
    algo = step_bytes_per_launch(cfg.n_steps, cfg.guidance_mode, cfg.d_latent, S)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    peak = peaks["hbm_gbs"]
    achieved = algo / (step_ms * 1e-3) / 1e9
    value = dist.world * frames_out / (ms_max * 1e-3)
    line = {
        "metric": "frames/s (img2img 512^2, 1-4 steps)",
        "value": round(value, 2),
        "unit": "frames/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic 512x512 u8 frames (moving gradients + noise, every frame processed)",
        "config": {
            "workload": (f"stream-batch pipeline, {S} streams/GPU x {cfg.n_steps}-step {cfg.guidance_mode}, "
                         "SSF eta 0.98 on, ANALYTIC denoiser (reference parity denoiser) + identity codec; "
                         "UNet/TAESD not built yet"),
            "streams_per_gpu": S, "n_steps": cfg.n_steps, "frame": "3x512x512 u8", "latent_elems": cfg.d_latent,
            "l2": "working set (latents %.0f MB/GPU) > 126 MB L2" % (S * cfg.n_steps * cfg.d_latent * 16 / 1e6),
        },
        "roofline": {"bound": "hbm", "kernel": "step_kernel (fused denoise+R-CFG+LCM update)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None,
                     "algo_bytes_per_launch": algo, "avg_launch_ms": round(step_ms, 5),
                     "ssf_avg_launch_ms": round(ssf_ms, 5),
                     "ssf_achieved_gbs": round(2 * FRAME_BYTES * S / (ssf_ms * 1e-3) / 1e9, 1) if ssf_ms else None,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)"},
        "e2e": {"value": round(dist.world * got / e2e_max, 2), "unit": "frames/s",
                "h2d_bytes_per_step": S * FRAME_BYTES, "d2h_bytes_per_step": S * cfg.d_latent * 4},
        "gpu_launches": kt["launches"],
        "clocks": clk.summary(),
    }
    p.close()
    return line


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the reference compiled from its own sources)
# ---------------------------------------------------------------------------

def _cpu_worker(a):
    nframes, d, n, guidance, seed = a
    from oracle.oracle import load, make_cfg

    o = load("ref") if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libstagger_ref.so")) else load("orc")
    rng = np.random.default_rng(seed)
    fr = rng.integers(0, 256, (nframes, d)).astype(np.float64)
    neg = o.gaussian(o.derive_seed(seed, 5), d) if guidance in ("cfg", "onetime_negative") else None
    cfg = make_cfg(n_steps=n, guidance_mode=guidance, ssf_enabled=True, eta=0.98, seed=seed, d_latent=d)
    t = time.perf_counter()
    r = o.run_pipeline(cfg, fr, neg=neg, want_payload=False)
    return len(r.seq), time.perf_counter() - t, o.which


def cpu_reference(args, seconds: float, steps: int = 1, warmup: int = 0):
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    d = FRAME_BYTES
    # calibrate: one short run on one core
    n_f, dt, which = _cpu_worker((args.n_steps + 2, d, args.n_steps, args.guidance, 0))
    per_frame = dt / n_f
    frames = max(args.n_steps + 1, int(seconds / per_frame / max(1, steps)))
    ctx = mp.get_context("fork")
    vals = []
    with ctx.Pool(cores) as pool:
        for i in range(warmup + steps):
            t = time.perf_counter()
            res = pool.map(_cpu_worker, [(frames, d, args.n_steps, args.guidance, 7 + c) for c in range(cores)])
            el = time.perf_counter() - t
            if i >= warmup:
                vals.append(sum(r[0] for r in res) / el)
    v = float(np.mean(vals))
    return {"value": round(v, 3), "unit": "frames/s", "cores": cores,
            "kind": "reference" if which == "ref" else "port",
            "sample": (f"{cores} processes x {frames} frames of 3x512x512 (as fp64 payload, identity codec), "
                       f"run_pipeline deterministic, n={args.n_steps} {args.guidance}, SSF on, analytic denoiser")}


def main():
    args = parse()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        steps = max(1, args.steps)
        warm = max(0, min(args.warmup, 1))
        budget = min(20.0, 150.0 / (steps + warm))
        cb = cpu_reference(args, budget * steps, steps=steps, warmup=warm)
        line = {"impl": "reference", "metric": "frames/s (img2img 512^2, 1-4 steps)", "value": cb["value"],
                "unit": "frames/s", "n_gpus": 0, "steps": steps, "warmup": warm, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": cb["sample"]}, "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    dist = Dist("nccl" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "none")
    line = run_ours(args, dist)
    if dist.rank == 0:
        if not args.no_cpu_baseline and dist.world == 1:
            line["cpu_baseline"] = cpu_reference(args, args.cpu_seconds)
        print(json.dumps(line))
    dist.close()


if __name__ == "__main__":
    main()
