#!/usr/bin/env python3
"""Benchmark of the B200 streaming denoise loop (contract: DESIGN.md §Measurement).

Headline workload (BASELINE.json configs[1]): img2img Stream Batch with 4
denoising steps (4 in-flight latents per stream) and TAESD encode/decode of
3x512x512 frames, random-init SD-2.1/SD-turbo-class UNet, on one B200.

One step = one pipeline iteration of every stream: push one u8 frame per
stream through the device SSF gate, TAESD encode, one batched UNet call over
all in-flight rows, the fused R-CFG / LCM step kernel and TAESD decode.
`value` = output frames/s with the input frames resident in HBM; `e2e` = the
same through the public C-ABI (sdx_pipeline_push) from pinned host frames,
with the H2D of the frames and the D2H of the decoded frames in the timed
region.  Multi-GPU: one process per GPU (torchrun), independent streams per
GPU, no collective on the data path; time = max over ranks (weak scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import glob
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
LATENT = 4 * 64 * 64


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=40)
    p.add_argument("--warmup", type=int, default=8)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--streams", type=int, default=1, help="independent streams per GPU")
    p.add_argument("--n-steps", type=int, default=4, help="denoising steps (in-flight frames per stream)")
    p.add_argument("--guidance", default="none")
    p.add_argument("--denoiser", choices=["unet", "analytic"], default="unet")
    p.add_argument("--no-ssf", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="launch every kernel eagerly instead of one CUDA graph per step")
    p.add_argument("--scene", choices=["dynamic", "near-static"], default="dynamic",
                   help="synthetic input: moving scene (SSF never skips) or a near-static one (SSF skips)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--profile-window", action="store_true",
                   help="cudaProfilerStart/Stop around the timed resident loop (ncu --profile-from-start off)")
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
                torch.cuda.set_device(int(os.environ.get("SDX_BENCH_DEVICE", self.local)))
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

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(r[0]) for r in self.rows if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        pw = [num(r[2]) for r in self.rows if len(r) > 2 and num(r[2]) is not None]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": num(self.rows[0][1]),
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def synthetic_frames(rng, n_iter, S):
    """Dynamic 512x512 RGB scenes (moving gradients + noise): the cosine to the
    previous frame stays well below eta, so every frame is processed while the
    gate still runs its full reduction."""
    yy, xx = np.mgrid[0:H, 0:W]
    out = np.empty((n_iter, S, FRAME_BYTES), dtype=np.uint8)
    for i in range(n_iter):
        for s in range(S):
            img = np.stack([(xx * (1 + s) + 13 * i) % 256, (yy * (2 + s) + 7 * i) % 256,
                            rng.integers(0, 256, (H, W))], -1)
            out[i, s] = img.astype(np.uint8).reshape(-1)
    return out


def near_static_frames(rng, n_iter, S):
    """A fixed 512x512 scene with sparse sensor noise (about 2% of the bytes
    redrawn per frame): cosines to the reference sit between eta = 0.98 and 1,
    so the similarity filter skips a share of the frames."""
    base = synthetic_frames(rng, 1, S)[0]
    out = np.empty((n_iter, S, FRAME_BYTES), dtype=np.uint8)
    for i in range(n_iter):
        for s in range(S):
            f = base[s].copy()
            idx = rng.integers(0, FRAME_BYTES, FRAME_BYTES // 50)
            f[idx] = rng.integers(0, 256, idx.size, dtype=np.uint8)
            out[i, s] = f
    return out


def workload_cfg(args):
    from paper_2312_12491_b200 import stagger as sg

    unet = args.denoiser == "unet"
    d = LATENT if unet else FRAME_BYTES
    neg = None
    if args.guidance in ("cfg", "onetime_negative"):
        neg = sg.sample_gaussian(sg.derive_seed(0, 5), d)
    return sg.EngineConfig(n_steps=args.n_steps, guidance_mode=args.guidance, gamma=1.4, delta=1.0,
                           ssf_enabled=not args.no_ssf, eta=0.98, seed=0, d_latent=d, negative_condition=neg,
                           backend="unet" if unet else "analytic", codec="taesd" if unet else "identity")


def rows_per_frame(n, guidance):
    return {"cfg": 2 * n, "onetime_negative": n + 1}.get(guidance, n)


def run_ours(args, dist: Dist):
    import ctypes as C

    from paper_2312_12491_b200 import _lib as L
    from paper_2312_12491_b200 import stagger as sg

    # SDX_BENCH_DEVICE pins every rank to one GPU (a smoke test of the N > 1 path on a one-GPU
    # box; the value is then not a scaling number)
    dev = int(os.environ.get("SDX_BENCH_DEVICE", dist.local))
    S = args.streams
    cfg = workload_cfg(args)
    ring = 4
    rng = np.random.default_rng(1000 + dist.rank)
    frames = (near_static_frames if args.scene == "near-static" else synthetic_frames)(rng, ring, S)
    p = sg.Pipeline(cfg, S, FRAME_BYTES, ring_depth=ring, device=dev, graph=not args.no_graph)
    unet_flops, codec_flops = p.flops()

    # ---- value: inputs resident in HBM ----
    p.upload_resident(frames)
    for _ in range(args.warmup):
        p.push_resident(copy_outputs=False)
    p.sync()
    # per-stage device times from an eager, event-bracketed pass (roofline inputs)
    p.set_profile(True)
    for _ in range(min(args.steps, 10)):
        p.push_resident(copy_outputs=False)
    p.sync()
    stages = p.stage_times()
    # timed pass: one CUDA graph per iteration (no per-kernel host launches)
    p.set_profile(False)
    for _ in range(2):
        p.push_resident(copy_outputs=False)
    p.sync()
    p.set_profile(False)
    dist.barrier()
    with Clocks(dev) as clk:
        p.sync()
        p.reset_timer()
        if args.profile_window:
            L.lib.sdx_profiler_start()
        for _ in range(args.steps):
            p.push_resident(copy_outputs=False)
        ms = p.device_time_ms()
        if args.profile_window:
            L.lib.sdx_profiler_stop()
        p.sync()
    stages["launches"] = p.stage_times()["launches"]
    skip_rate = float(np.mean([p.report(s)["skip_rate"] for s in range(S)]))
    ms_max = dist.max(ms)
    frames_out = args.steps * S  # steady state: every stream emits one frame per iteration

    # ---- e2e: public API from pinned host frames, decoded frames copied back ----
    hp = C.c_void_p()
    nbytes = frames.nbytes
    assert L.lib.sdx_host_alloc(nbytes, C.byref(hp)) == 0
    host = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(hp.value)).reshape(frames.shape)
    host[:] = frames
    p.close()
    q = sg.Pipeline(cfg, S, FRAME_BYTES, ring_depth=ring, device=dev, graph=not args.no_graph)
    for i in range(args.warmup):
        q.push_ptr(hp.value + (i % ring) * S * FRAME_BYTES)
        for s in range(S):
            q.pop_all(s)
    q.sync()
    for s in range(S):
        q.pop_all(s)
    dist.barrier()
    got = 0
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

    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {}
    it = max(1, stages["iterations"])
    rpf = rows_per_frame(cfg.n_steps, cfg.guidance_mode)
    value = dist.world * frames_out / (ms_max * 1e-3)
    if args.denoiser == "unet":
        den_ms = stages["denoiser"] / it
        algo = S * rpf * unet_flops  # FLOPs of one batched UNet call (steady state)
        achieved = algo / (den_ms * 1e-3) / 1e12
        peak = peaks.get("bf16_tflops_sustained", 1400.0)
        traffic, traffic_detail = None, None  # DRAM bytes of one UNet forward at this row count (ncu capture)
        for tf in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_unet_traffic.json"))):
            td = json.load(open(tf))
            if td.get("rows") == S * rpf:
                traffic = td["dram_bytes"]
                traffic_detail = {"read": td["dram_bytes_read"], "write": td["dram_bytes_write"],
                                  "source": os.path.relpath(tf, ROOT)}
        roof = {"bound": "tensor", "kernel": "UNet forward (tcgen05 conv/GEMM + flash-attention kernels), "
                                              f"{S * rpf} rows/launch",
                "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_detail": traffic_detail, "algo_flops_per_launch": algo,
                "avg_launch_ms": round(den_ms, 4),
                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS, long loop)"}
        frame_flops = rpf * unet_flops + codec_flops
        workload = (f"img2img Stream Batch, {S} stream(s)/GPU x {cfg.n_steps}-step {cfg.guidance_mode}, "
                    f"TAESD enc/dec 512x512, random-init SD-2.1/SD-turbo UNet (bf16, fp32 accum), "
                    f"SSF eta 0.98 {'on' if cfg.ssf_enabled else 'off'}")
        d2h = S * FRAME_BYTES
    else:
        den_ms = stages["step"] / it
        algo = None
        roof = {"bound": "hbm", "kernel": "fused step kernel", "achieved": None,
                "peak": peaks.get("hbm_gbs", 6536.4), "unit": "GB/s", "frac": None, "traffic": None}
        frame_flops = None
        workload = f"analytic-denoiser pipeline, {S} streams x {cfg.n_steps} steps, identity codec"
        d2h = S * cfg.d_latent * 4
    line = {
        "metric": "frames/s (img2img 512^2, 1-4 steps)",
        "value": round(value, 3),
        "unit": "frames/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16" if args.denoiser == "unet" else "f32",
        "data": ("synthetic 512x512 u8 frames (%s), random-init UNet/TAESD weights"
                 % ("moving gradients + noise" if args.scene == "dynamic" else "near-static scene + sparse noise")),
        "config": {
            "workload": workload, "streams_per_gpu": S, "n_steps": cfg.n_steps, "guidance": cfg.guidance_mode,
            "rows_per_tick": S * rpf, "frame": "3x512x512 u8", "latent": "4x64x64", "scene": args.scene,
            "ssf_skip_rate": round(skip_rate, 4),
            "gflop_per_frame": round(frame_flops / 1e9, 1) if frame_flops else None,
            "l2": "per-step working set (UNet activations ~%.1f GB) exceeds the 126 MB L2" % (
                S * rpf * 0.25 if args.denoiser == "unet" else 0.4),
        },
        "roofline": roof,
        "stage_ms_per_step": {k: round(stages[k] / it, 4) for k in sg.Pipeline.STAGES},
        "e2e": {"value": round(dist.world * got / e2e_max, 3), "unit": "frames/s",
                "h2d_bytes_per_step": S * FRAME_BYTES, "d2h_bytes_per_step": d2h},
        "gpu_launches": stages["launches"],
        "clocks": clk.summary(),
    }
    if frame_flops:
        line["model_tflops"] = round(frame_flops * frames_out / (ms * 1e-3) / 1e12, 2)
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
    """The reference's own CPU path (run_pipeline, analytic denoiser: it has no
    UNet or TAESD) on the same 3x512x512 frames, one stream per host core."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    d = FRAME_BYTES
    n_f, dt, which = _cpu_worker((args.n_steps + 2, d, args.n_steps, args.guidance, 0))
    per_frame = dt / n_f
    frames = max(args.n_steps + 1, int(seconds / per_frame / max(1, steps)))
    ctx = mp.get_context("fork")
    vals = []
    els = []
    with ctx.Pool(cores) as pool:
        for i in range(warmup + steps):
            # warm-up steps run a short sample (they only warm the pool and caches)
            nf = frames if i >= warmup else max(args.n_steps + 1, frames // 8)
            t = time.perf_counter()
            res = pool.map(_cpu_worker, [(nf, d, args.n_steps, args.guidance, 7 + c) for c in range(cores)])
            el = time.perf_counter() - t
            if i >= warmup:
                vals.append(sum(r[0] for r in res) / el)
                els.append(el)
    v = float(np.mean(vals))
    return {"value": round(v, 3), "unit": "frames/s", "cores": cores, "ms_per_step": 1e3 * float(np.mean(els)),
            "kind": "reference" if which == "ref" else "port",
            "sample": (f"{cores} processes x {frames} frames of 3x512x512 (fp64 payload, identity codec: the "
                       f"reference has no UNet/TAESD), run_pipeline deterministic, n={args.n_steps} {args.guidance}, "
                       "SSF on, analytic denoiser")}


def main():
    args = parse()
    if os.environ.get("SDX_ABLATE"):
        # op-skipping timing ablation (unet.cu): never a bench number
        sys.exit("bench.py: SDX_ABLATE is set (skips UNet ops); unset it to measure")
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        steps = max(1, args.steps)
        warm = max(0, args.warmup)
        budget = min(20.0, 150.0 / (steps + warm / 8.0))  # CPU seconds per timed step (warm-up steps: 1/8)
        cb = cpu_reference(args, budget * steps, steps=steps, warmup=warm)
        ms_step = cb.pop("ms_per_step")
        # the same workload shape as our arm's line (streams, steps, guidance, frames); the
        # reference computes it with its own analytic denoiser and identity codec (it has no
        # UNet or TAESD), one stream per host core
        config = {"workload": (f"img2img Stream Batch, {args.streams} stream(s) x {args.n_steps}-step "
                               f"{args.guidance}, 3x512x512 frames, SSF eta 0.98 "
                               f"{'off' if args.no_ssf else 'on'}: the reference's CPU run_pipeline"),
                  "streams_per_gpu": args.streams, "n_steps": args.n_steps, "guidance": args.guidance,
                  "frame": "3x512x512 u8", "reference_denoiser": "analytic Gaussian model (no UNet in the reference)",
                  "reference_codec": "identity (no TAESD in the reference)", "host_streams": cb["cores"]}
        line = {"impl": "reference", "metric": "frames/s (img2img 512^2, 1-4 steps)", "value": cb["value"],
                "unit": "frames/s", "n_gpus": 0, "steps": steps, "warmup": warm, "ms_per_step": round(ms_step, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config, "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    dist = Dist(os.environ.get("SDX_BENCH_DIST_BACKEND", "nccl") if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "none")
    line = run_ours(args, dist)
    if dist.rank == 0:
        if not args.no_cpu_baseline and dist.world == 1:
            cb = cpu_reference(args, args.cpu_seconds)
            cb.pop("ms_per_step", None)
            line["cpu_baseline"] = cb
        print(json.dumps(line))
    dist.close()


if __name__ == "__main__":
    main()
