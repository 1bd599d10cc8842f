"""Python mirror of the reference `stagger` operator API over the sm_100a
C-ABI (include/stagger_b200.h).

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/core/include/stagger/*.hpp):

==========================  =============================================
this module                 reference
==========================  =============================================
EngineConfig                EngineConfig (core.hpp:41-69)
build_schedule              build_schedule (schedule.cpp:29-58)
derive_seed / sample_gaussian  rng.cpp:7-20
build_precompute            build_precompute (precompute.cpp:7-21)
StreamBatchEngine           StreamBatchEngine (engine.hpp:58-97)
SsfState                    SsfState (ssf.hpp:25-42)
run_pipeline / Pipeline     run_pipeline deterministic mode (pipeline.cpp:152-214)
InvalidArgument/LogicError/
StaggerRuntimeError         std::invalid_argument / logic_error / runtime_error
==========================  =============================================

All numerics run on the GPU through libstagger_b200.so; this module only
marshals arguments.  Nothing here calls a CPU implementation of the path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L

kStreamNoiseCache, kStreamSsf, kStreamSource, kStreamCondition = 1, 2, 3, 4


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class LogicError(RuntimeError):
    """std::logic_error"""


class StaggerRuntimeError(RuntimeError):
    """std::runtime_error"""


class CudaError(RuntimeError):
    pass


class Unsupported(NotImplementedError):
    pass


_EXC = {L.SDX_INVALID_ARGUMENT: InvalidArgument, L.SDX_LOGIC_ERROR: LogicError,
        L.SDX_RUNTIME_ERROR: StaggerRuntimeError, L.SDX_CUDA_ERROR: CudaError, L.SDX_UNSUPPORTED: Unsupported}


def _check(st: int, err=None):
    if st != L.SDX_OK:
        msg = (err or L.lib.sdx_last_error)()
        raise _EXC.get(st, RuntimeError)(msg.decode() if msg else f"status {st}")


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a, n=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.size != n:
        raise InvalidArgument(f"length {a.size} != {n}")
    return a


# ---------------------------------------------------------------------------
# config / schedule / precompute
# ---------------------------------------------------------------------------

@dataclass
class EngineConfig:
    n_steps: int = 4
    guidance_mode: str = "none"
    gamma: float = 1.4
    delta: float = 1.0
    ssf_enabled: bool = False
    eta: float = 0.98
    seed: int = 0
    cross_frame_attention: bool = False
    d_latent: int = 8
    t_grid: int = 1000
    entry_strength: float = 1.0
    backend: str = "analytic"
    data_variance: float = 1.0
    lcm_mode: str = "exact"
    codec: str = "identity"
    queue_capacity: int = 8
    condition: Optional[np.ndarray] = None
    negative_condition: Optional[np.ndarray] = None

    def to_c(self) -> L.sdx_config:
        if self.guidance_mode not in L.GUIDANCE:
            raise InvalidArgument(f"unknown guidance_mode: {self.guidance_mode}")
        return L.sdx_config(self.n_steps, L.GUIDANCE[self.guidance_mode], self.gamma, self.delta,
                            int(self.ssf_enabled), self.eta, self.seed, int(self.cross_frame_attention),
                            self.d_latent, self.t_grid, self.entry_strength, L.BACKEND.get(self.backend, -1),
                            self.data_variance, L.LCM.get(self.lcm_mode, -1), L.CODEC.get(self.codec, -1),
                            self.queue_capacity)


@dataclass
class ScheduleStep:
    tau: int
    alpha: float
    beta: float

    def is_terminal(self):
        return self.beta == 0.0


def derive_seed(seed: int, tag: int) -> int:
    return L.lib.sdx_derive_seed(seed, tag)


def sample_gaussian(seed: int, d: int) -> np.ndarray:
    out = np.empty(d)
    _check(L.lib.sdx_sample_gaussian(seed, d, _dp(out)), L.lib.sdx_precompute_error)
    return out


def build_schedule(n: int, t_grid: int = 1000, entry_strength: float = 1.0) -> list[ScheduleStep]:
    buf = (L.sdx_step * max(n, 1))()
    _check(L.lib.sdx_build_schedule(n, t_grid, entry_strength, buf), L.lib.sdx_precompute_error)
    return [ScheduleStep(s.tau, s.alpha, s.beta) for s in buf[:n]]


@dataclass
class PrecomputeCache:
    schedule: list
    eps_cached: np.ndarray  # n x d
    lcm_mode: str = "exact"
    cond_embeddings: dict = field(default_factory=dict)

    def steps_c(self):
        arr = (L.sdx_step * len(self.schedule))()
        for i, s in enumerate(self.schedule):
            arr[i] = L.sdx_step(s.tau, s.alpha, s.beta)
        return arr


def build_precompute(cfg: EngineConfig, conditions: dict | None = None) -> PrecomputeCache:
    sched = build_schedule(cfg.n_steps, cfg.t_grid, cfg.entry_strength)
    eps = np.empty((cfg.n_steps, cfg.d_latent))
    _check(L.lib.sdx_build_noise_cache(cfg.seed, cfg.n_steps, cfg.d_latent, _dp(eps)), L.lib.sdx_precompute_error)
    return PrecomputeCache(sched, eps, cfg.lcm_mode, dict(conditions or {}))


def resolve_condition(cfg: EngineConfig) -> np.ndarray:
    """pipeline.cpp:30-34: explicit condition or Rng(derive_seed(seed, 4)) draws."""
    if cfg.condition is not None:
        return _f64(cfg.condition, cfg.d_latent)
    return sample_gaussian(derive_seed(cfg.seed, kStreamCondition), cfg.d_latent)


# ---------------------------------------------------------------------------
# StreamBatchEngine
# ---------------------------------------------------------------------------

@dataclass
class EmittedFrame:
    seq_id: int
    x0_hat: np.ndarray
    ingest_tick: int
    emit_tick: int


@dataclass
class TickResult:
    emitted: Optional[EmittedFrame]
    denoiser_calls: int
    element_evals: int


class StreamBatchEngine:
    """engine.hpp:58-97 on the device: one fused kernel pass per tick."""

    def __init__(self, cfg: EngineConfig, cache: PrecomputeCache | None = None, device: int = 0):
        self.cfg = cfg
        self.cache = cache or build_precompute(cfg)
        self.d = cfg.d_latent
        self._h = C.c_void_p()
        c = cfg.to_c()
        c.lcm_mode = L.LCM.get(self.cache.lcm_mode, -1)
        eps = _f64(self.cache.eps_cached)
        if eps.shape != (len(self.cache.schedule), cfg.d_latent):
            raise InvalidArgument("StreamBatchEngine: noise cache length != n_steps")
        neg = cfg.negative_condition
        negp = _dp(_f64(neg, cfg.d_latent)) if neg is not None else None
        self._neg_keep = neg
        _check(L.lib.sdx_engine_create(C.byref(c), self.cache.steps_c(), len(self.cache.schedule), _dp(eps), negp,
                                       device, C.byref(self._h)))
        self._out = np.empty(self.d)

    def close(self):
        if self._h and self._h.value:
            L.lib.sdx_engine_destroy(self._h)
            self._h = C.c_void_p()

    __del__ = close

    def ingest(self, seq_id: int, x0, cond) -> None:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        emb = cond if isinstance(cond, np.ndarray) or not hasattr(cond, "embedding") else cond.embedding
        emb = np.ascontiguousarray(emb, dtype=np.float64)
        if x0.size != self.d:
            raise InvalidArgument("ingest: latent length != d_latent")
        if emb.size != self.d:
            raise InvalidArgument("ingest: condition embedding length != d_latent")
        _check(L.lib.sdx_engine_ingest(self._h, seq_id, _dp(x0), _dp(emb)))

    def tick(self) -> TickResult:
        r = L.sdx_tick_result()
        out = np.empty(self.d)
        _check(L.lib.sdx_engine_tick(self._h, C.byref(r), _dp(out)))
        em = None
        if r.emitted_seq >= 0:
            em = EmittedFrame(r.emitted_seq, out, r.ingest_tick, r.emit_tick)
        return TickResult(em, r.denoiser_calls, r.element_evals)

    def ticks_completed(self) -> int:
        v = C.c_int64()
        _check(L.lib.sdx_engine_ticks_completed(self._h, C.byref(v)))
        return v.value

    def inflight_size(self) -> int:
        v = C.c_int()
        _check(L.lib.sdx_engine_inflight(self._h, C.byref(v)))
        return v.value

    def idle(self) -> bool:
        return self.inflight_size() == 0

    def step_indices(self) -> list[int]:
        buf = (C.c_int * max(1, self.cfg.n_steps + 1))()
        n = C.c_int()
        _check(L.lib.sdx_engine_step_indices(self._h, buf, C.byref(n)))
        return list(buf[: n.value])

    def min_inflight_seq(self) -> Optional[int]:
        v = C.c_int64()
        _check(L.lib.sdx_engine_min_inflight_seq(self._h, C.byref(v)))
        return None if v.value == 2**63 - 1 else v.value

    def counters(self) -> tuple[int, int]:
        a, b = C.c_uint64(), C.c_uint64()
        _check(L.lib.sdx_engine_counters(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def reset_counters(self):
        _check(L.lib.sdx_engine_reset_counters(self._h))

    def last_tick_ms(self) -> float:
        v = C.c_float()
        _check(L.lib.sdx_engine_last_tick_ms(self._h, C.byref(v)))
        return v.value


# ---------------------------------------------------------------------------
# SsfState
# ---------------------------------------------------------------------------

class SsfState:
    """ssf.hpp:25-42 on the device; frames are u8 payloads of frame_bytes."""

    def __init__(self, eta: float, rng_seed: int, frame_bytes: int, max_skip: int = 0, device: int = 0):
        self._h = C.c_void_p()
        self.frame_bytes = frame_bytes
        _check(L.lib.sdx_ssf_create(eta, rng_seed, max_skip, frame_bytes, device, C.byref(self._h)))

    def close(self):
        if self._h and self._h.value:
            L.lib.sdx_ssf_destroy(self._h)
            self._h = C.c_void_p()

    __del__ = close

    def gate_many(self, frames: np.ndarray, with_sims: bool = False):
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        nf = frames.shape[0] if frames.ndim > 1 else 1
        if frames.size != nf * self.frame_bytes:
            raise InvalidArgument("cosine_similarity: dimension mismatch")
        dec = np.empty(nf, dtype=np.int32)
        sims = np.empty(nf) if with_sims else None
        _check(L.lib.sdx_ssf_gate(self._h, frames.ctypes.data, nf, dec.ctypes.data_as(C.POINTER(C.c_int)),
                                  _dp(sims) if sims is not None else None))
        return (dec, sims) if with_sims else dec

    def gate(self, frame) -> str:
        return "skip" if self.gate_many(np.asarray(frame)[None])[0] == 1 else "process"

    def counters(self):
        a, b = C.c_uint64(), C.c_uint64()
        _check(L.lib.sdx_ssf_counters(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def examined(self):
        return self.counters()[0]

    def skipped(self):
        return self.counters()[1]


# ---------------------------------------------------------------------------
# Pipeline
# ---------------------------------------------------------------------------

class Pipeline:
    """S independent streams, one batched device tick per push (run_pipeline
    deterministic mode per stream, pipeline.cpp:152-214)."""

    def __init__(self, cfg: EngineConfig, n_streams: int = 1, frame_bytes: int | None = None,
                 max_skip: int = 0, ring_depth: int = 4, seeds=None, conds=None, negs=None, device: int = 0,
                 graph: bool = False):
        self.cfg = cfg
        self.S = n_streams
        self.D = frame_bytes if frame_bytes is not None else cfg.d_latent
        self.d = cfg.d_latent
        seeds = list(seeds) if seeds is not None else [cfg.seed + s for s in range(n_streams)]
        steps = None
        eps = np.empty((n_streams, cfg.n_steps, cfg.d_latent))
        cond = np.empty((n_streams, cfg.d_latent))
        for s, sd in enumerate(seeds):
            scfg = EngineConfig(**{**cfg.__dict__, "seed": sd})
            pc = build_precompute(scfg)
            steps = pc.steps_c()
            eps[s] = pc.eps_cached
            cond[s] = conds[s] if conds is not None else resolve_condition(scfg)
        neg = None
        if negs is not None:
            neg = _f64(negs).reshape(n_streams, cfg.d_latent)
        elif cfg.negative_condition is not None:
            neg = np.tile(_f64(cfg.negative_condition, cfg.d_latent), (n_streams, 1))
        # The drop-in stream seed ordering: stream s uses seed base+s.
        pc_cfg = L.sdx_pipeline_config(cfg.to_c(), n_streams, self.D, max_skip, ring_depth, int(graph))
        self._seed_check = seeds
        if any(sd != cfg.seed + i for i, sd in enumerate(seeds)):
            raise InvalidArgument("Pipeline: stream seeds must be cfg.seed + stream index")
        self._h = C.c_void_p()
        self._keep = (eps, cond, neg)
        _check(L.lib.sdx_pipeline_create(C.byref(pc_cfg), steps, _dp(eps), _dp(cond),
                                         _dp(neg) if neg is not None else None, device, C.byref(self._h)))
        self.out_is_u8 = cfg.codec == "taesd"
        self.out_bytes = self.D if self.out_is_u8 else 4 * self.d

    def close(self):
        if self._h and self._h.value:
            L.lib.sdx_pipeline_destroy(self._h)
            self._h = C.c_void_p()

    __del__ = close

    def push(self, frames: np.ndarray, seq_ids=None):
        """One iteration over the S streams' frames.  seq_ids (S source sequence ids,
        pipeline.cpp:176) default to the frame index."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        if frames.size != self.S * self.D:
            raise InvalidArgument("LatentCodec::encode: dim mismatch")
        if seq_ids is None:
            _check(L.lib.sdx_pipeline_push(self._h, frames.ctypes.data))
        else:
            ids = np.ascontiguousarray(np.broadcast_to(np.asarray(seq_ids, dtype=np.int64), (self.S,)))
            _check(L.lib.sdx_pipeline_push_seq(self._h, frames.ctypes.data, ids.ctypes.data))

    def tick(self) -> bool:
        """A frame-less iteration (tick without ingest) unless every stream is idle."""
        ran = C.c_int()
        _check(L.lib.sdx_pipeline_tick(self._h, C.byref(ran)))
        return bool(ran.value)

    def idle(self) -> bool:
        v = C.c_int()
        _check(L.lib.sdx_pipeline_idle(self._h, C.byref(v)))
        return bool(v.value)

    def push_ptr(self, ptr: int):
        _check(L.lib.sdx_pipeline_push(self._h, C.c_void_p(ptr)))

    def upload_resident(self, frames: np.ndarray):
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        _check(L.lib.sdx_pipeline_upload_resident(self._h, frames.ctypes.data, frames.shape[0]))

    def push_resident(self, copy_outputs: bool = False):
        _check(L.lib.sdx_pipeline_push_resident(self._h, int(copy_outputs)))

    def finish(self):
        _check(L.lib.sdx_pipeline_finish(self._h))

    def sync(self):
        _check(L.lib.sdx_pipeline_sync(self._h))

    def pop_all(self, stream: int):
        out = []
        seq, has = C.c_int64(), C.c_int()
        while True:
            buf = np.empty(self.out_bytes, dtype=np.uint8)  # popped into directly (one host copy)
            _check(L.lib.sdx_pipeline_pop(self._h, stream, C.byref(seq), buf.ctypes.data, C.byref(has)))
            if not has.value:
                return out
            out.append((seq.value, buf if self.out_is_u8 else buf.view(np.float32)))

    def report(self, stream: int = 0) -> dict:
        r = L.sdx_report()
        _check(L.lib.sdx_pipeline_report(self._h, stream, C.byref(r)))
        d = {k: getattr(r, k) for k, _ in L.sdx_report._fields_}
        d["incomplete"] = bool(d["incomplete"])
        d["error"] = L.lib.sdx_pipeline_error_message(self._h, stream).decode()
        d["mode"] = "deterministic"
        return d

    def decisions(self, stream: int = 0) -> np.ndarray:
        n = C.c_int()
        _check(L.lib.sdx_pipeline_decisions(self._h, stream, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=np.int32)
        _check(L.lib.sdx_pipeline_decisions(self._h, stream, out.ctypes.data_as(C.POINTER(C.c_int)), n.value,
                                            C.byref(n)))
        return out

    def trace(self, stream: int = 0) -> list[dict]:
        """Per-tick log (TickLogEntry, engine.hpp:43-50) of one stream: tick, ingested /
        emitted sequence ids (None for no frame), denoiser calls / element evals, and the
        iteration's device time (ns, 0 unless stage profiling is on)."""
        n = C.c_int()
        _check(L.lib.sdx_pipeline_trace(self._h, stream, None, 0, C.byref(n)))
        buf = (L.sdx_trace_entry * max(1, n.value))()
        _check(L.lib.sdx_pipeline_trace(self._h, stream, buf, n.value, C.byref(n)))
        out = []
        for e in buf[:n.value]:
            out.append({"tick": e.tick, "ingested": None if e.ingested < 0 else e.ingested,
                        "emitted": None if e.emitted < 0 else e.emitted, "calls": e.calls,
                        "element_evals": e.element_evals, "elapsed_ns": e.elapsed_ns})
        return out

    def reset_timer(self):
        _check(L.lib.sdx_pipeline_reset_timer(self._h))

    def set_profile(self, on: bool = True):
        _check(L.lib.sdx_pipeline_set_profile(self._h, int(on)))

    STAGES = ("ssf", "control", "encode", "denoiser", "step", "decode")

    def stage_times(self) -> dict:
        """Summed device ms per pipeline stage since set_profile(True), plus
        iterations and library kernel launches."""
        ms = (C.c_double * 6)()
        it, nl = C.c_int64(), C.c_int64()
        _check(L.lib.sdx_pipeline_stage_times(self._h, ms, C.byref(it), C.byref(nl)))
        d = {k: ms[i] for i, k in enumerate(self.STAGES)}
        d["iterations"] = it.value
        d["launches"] = nl.value
        return d

    def flops(self) -> tuple[float, float]:
        a, b = C.c_double(), C.c_double()
        _check(L.lib.sdx_pipeline_flops(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def device_time_ms(self) -> float:
        v = C.c_float()
        _check(L.lib.sdx_pipeline_device_time_ms(self._h, C.byref(v)))
        return v.value


def run_pipeline(cfg: EngineConfig, frames: np.ndarray, max_skip: int = 0, device: int = 0, seq_ids=None):
    """Deterministic run_pipeline over u8 frames [N, D] (vector_source order;
    seq = index unless seq_ids gives the source ids).  Returns (sink list of
    (seq, payload), report dict)."""
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    p = Pipeline(cfg, 1, frames.shape[1], max_skip=max_skip, device=device)
    sink = []
    try:
        for i, f in enumerate(frames):
            p.push(f, None if seq_ids is None else [seq_ids[i]])
            sink.extend(p.pop_all(0))
        p.finish()
        sink.extend(p.pop_all(0))
        return sink, p.report(0)
    finally:
        p.close()
