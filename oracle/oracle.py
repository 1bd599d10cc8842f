"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the two CPU checkers.

* ``load("orc")``: my plain-C restatement (oracle/stagger_oracle.c ->
  oracle/_build/liboracle.so).
* ``load("ref")``: the unmodified reference core compiled from
  /root/reference/proj/core/src (oracle/Makefile -> oracle/_ref/libstagger_ref.so).

Both expose the same entry points (prefix ``orc_`` / ``ref_``) so a test can run
the same scenario through either and compare.  Only tests/, the smoke check in
__graft_entry__.py and bench.py's CPU-baseline legs import this module; the
product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "orc": os.path.join(HERE, "_build", "liboracle.so"),
    "ref": os.path.join(HERE, "_ref", "libstagger_ref.so"),
}

GUIDANCE = {"none": 0, "cfg": 1, "self_negative": 2, "onetime_negative": 3}
LCM = {"exact": 0, "boundary_approx": 1}

D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)
U64 = C.POINTER(C.c_uint64)


class Cfg(C.Structure):
    """Plain-C mirror of stagger::EngineConfig's hot-path fields (core.hpp:41-69)."""

    _fields_ = [
        ("n_steps", C.c_int),
        ("guidance_mode", C.c_int),
        ("gamma", C.c_double),
        ("delta", C.c_double),
        ("ssf_enabled", C.c_int),
        ("eta", C.c_double),
        ("seed", C.c_uint64),
        ("d_latent", C.c_int),
        ("t_grid", C.c_int),
        ("entry_strength", C.c_double),
        ("data_variance", C.c_double),
        ("lcm_mode", C.c_int),
        ("codec", C.c_int),
        ("queue_capacity", C.c_int),
        ("cross_frame_attention", C.c_int),
    ]


class Report(C.Structure):
    _fields_ = [
        (n, C.c_uint64)
        for n in (
            "frames_in", "frames_out", "duplicates", "stale_skips", "input_drops",
            "output_drops", "ticks", "denoiser_calls", "element_evals", "ssf_examined",
            "ssf_skipped",
        )
    ] + [
        ("skip_rate", C.c_double),
        ("latency_ticks_mean", C.c_double),
        ("latency_ticks_min", C.c_int64),
        ("latency_ticks_max", C.c_int64),
        ("mean_frame_time_ms", C.c_double),
        ("throughput_fps", C.c_double),
        ("wall_ms", C.c_double),
        ("incomplete", C.c_int),
    ]


def make_cfg(n_steps=4, guidance_mode="none", gamma=1.4, delta=1.0, ssf_enabled=False,
             eta=0.98, seed=0, d_latent=8, t_grid=1000, entry_strength=1.0,
             data_variance=1.0, lcm_mode="exact", codec=0, queue_capacity=8,
             cross_frame_attention=False) -> Cfg:
    return Cfg(n_steps, GUIDANCE[guidance_mode] if isinstance(guidance_mode, str) else guidance_mode,
               gamma, delta, int(ssf_enabled), eta, seed, d_latent, t_grid, entry_strength,
               data_variance, LCM[lcm_mode] if isinstance(lcm_mode, str) else lcm_mode, codec,
               queue_capacity, int(cross_frame_attention))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _dp(a: np.ndarray):
    return a.ctypes.data_as(D)


class Oracle:
    def __init__(self, which: str):
        path = PATHS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        self.which = which
        self.p = which + "_"
        self.lib = C.CDLL(path)
        L = self.lib
        p = self.p
        self._f("last_error").restype = C.c_char_p
        self._f("derive_seed").restype = C.c_uint64
        self._f("derive_seed").argtypes = [C.c_uint64, C.c_uint64]
        self._f("rng_uniforms").argtypes = [C.c_uint64, C.c_int, D]
        self._f("rng_u64").argtypes = [C.c_uint64, C.c_int, U64]
        self._f("sample_gaussian").argtypes = [C.c_uint64, C.c_int, D]
        self._f("build_schedule").argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(C.c_int), D, D]
        self._f("lcm_coefficients").argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, D, D]
        self._f("cosine").restype = C.c_double
        self._f("cosine").argtypes = [D, D, C.c_int]
        self._f("skip_probability").restype = C.c_double
        self._f("skip_probability").argtypes = [C.c_double, C.c_double]
        self._f("engine_create").argtypes = [C.POINTER(Cfg), D, D, C.POINTER(C.c_void_p)]
        self._f("engine_destroy").argtypes = [C.c_void_p]
        self._f("engine_ingest").argtypes = [C.c_void_p, C.c_int64, D]
        self._f("engine_tick").argtypes = [C.c_void_p, I64, D, I64, I64, U64, U64]
        self._f("engine_idle").argtypes = [C.c_void_p]
        self._f("engine_ticks").argtypes = [C.c_void_p]
        self._f("engine_ticks").restype = C.c_int64
        self._f("engine_inflight").argtypes = [C.c_void_p]
        self._f("engine_min_inflight_seq").argtypes = [C.c_void_p]
        self._f("engine_min_inflight_seq").restype = C.c_int64
        self._f("engine_step_indices").argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        self._f("engine_counters").argtypes = [C.c_void_p, U64, U64]
        self._f("engine_eps_cached").argtypes = [C.c_void_p, C.c_int, D]
        self._f("sequential").argtypes = [C.POINTER(Cfg), D, D, D, D]
        self._f("ssf_destroy").argtypes = [C.c_void_p]
        self._f("ssf_gate").argtypes = [C.c_void_p, D, C.c_int]
        self._f("ssf_counters").argtypes = [C.c_void_p, U64, U64]
        self._f("stream_frames").argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, D]
        if which == "orc":
            self._f("ssf_create").argtypes = [C.c_double, C.c_uint64, C.c_int, C.POINTER(C.c_void_p)]
            self._f("run_pipeline").argtypes = [C.POINTER(Cfg), D, D, D, C.c_int, C.c_int, C.c_int,
                                                I64, D, C.c_int, C.POINTER(C.c_int),
                                                C.POINTER(C.c_int), C.POINTER(Report)]
        else:
            self._f("ssf_create").argtypes = [C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]
            self._f("run_pipeline").argtypes = [C.POINTER(Cfg), D, D, D, C.c_int, C.c_int, I64, D,
                                                C.c_int, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        del L, p

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, st):
        if st != 0:
            raise OracleError(st, self._f("last_error")().decode())

    # -- rng / schedule ---------------------------------------------------
    def derive_seed(self, seed, tag):
        return self._f("derive_seed")(seed, tag)

    def uniforms(self, seed, n):
        out = np.empty(n)
        self._f("rng_uniforms")(seed, n, _dp(out))
        return out

    def u64(self, seed, n):
        out = np.empty(n, dtype=np.uint64)
        self._f("rng_u64")(seed, n, out.ctypes.data_as(U64))
        return out

    def gaussian(self, seed, d):
        out = np.empty(d)
        self._check(self._f("sample_gaussian")(seed, d, _dp(out)))
        return out

    def schedule(self, n, t_grid=1000, entry=1.0):
        taus = (C.c_int * n)()
        a = np.empty(n)
        b = np.empty(n)
        self._check(self._f("build_schedule")(n, t_grid, entry, taus, _dp(a), _dp(b)))
        return list(taus), a, b

    def lcm(self, tau, alpha, beta, mode="exact"):
        cs, co = C.c_double(), C.c_double()
        self._f("lcm_coefficients")(tau, alpha, beta, LCM[mode], C.byref(cs), C.byref(co))
        return cs.value, co.value

    def cosine(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        return self._f("cosine")(_dp(a), _dp(b), len(a))

    def skip_probability(self, sim, eta):
        return self._f("skip_probability")(sim, eta)

    # -- engine -----------------------------------------------------------
    def engine(self, cfg: Cfg, cond, neg=None):
        return _Engine(self, cfg, cond, neg)

    def sequential(self, cfg: Cfg, cond, x0, neg=None):
        out = np.empty(cfg.d_latent)
        cond = np.ascontiguousarray(cond, dtype=np.float64)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        negp = _dp(np.ascontiguousarray(neg, dtype=np.float64)) if neg is not None else None
        self._check(self._f("sequential")(C.byref(cfg), _dp(cond), negp, _dp(x0), _dp(out)))
        return out

    # -- ssf --------------------------------------------------------------
    def ssf(self, eta, rng_seed, max_skip=0):
        return _Ssf(self, eta, rng_seed, max_skip)

    # -- pipeline ---------------------------------------------------------
    def run_pipeline(self, cfg: Cfg, frames: np.ndarray, cond=None, neg=None, max_skip=0,
                     want_payload=True):
        frames = np.ascontiguousarray(frames, dtype=np.float64)
        nf, d = frames.shape
        cap = nf * 2 + 8
        seq = np.empty(cap, dtype=np.int64)
        pay = np.empty((cap, cfg.d_latent)) if want_payload else None
        n_out = C.c_int()
        condp = _dp(np.ascontiguousarray(cond, dtype=np.float64)) if cond is not None else None
        negp = _dp(np.ascontiguousarray(neg, dtype=np.float64)) if neg is not None else None
        payp = _dp(pay) if pay is not None else None
        if self.which == "orc":
            rep = Report()
            dec = np.empty(nf, dtype=np.int32)
            self._check(self._f("run_pipeline")(
                C.byref(cfg), condp, negp, _dp(frames), nf, d, max_skip, seq.ctypes.data_as(I64),
                payp, cap, C.byref(n_out), dec.ctypes.data_as(C.POINTER(C.c_int)), C.byref(rep)))
            report = {k: getattr(rep, k) for k, _ in Report._fields_}
            report["incomplete"] = bool(report["incomplete"])
        else:
            if max_skip > 0:
                raise ValueError("the reference has no max_skip (SURVEY §8c)")
            buf = C.create_string_buffer(1 << 14)
            self._check(self._f("run_pipeline")(
                C.byref(cfg), condp, negp, _dp(frames), nf, d, seq.ctypes.data_as(I64), payp, cap,
                C.byref(n_out), buf, len(buf)))
            import json
            report = json.loads(buf.value.decode())
            dec = None
        n = n_out.value
        return PipelineResult(seq[:n].copy(), pay[:n].copy() if pay is not None else None, report, dec)

    def stream_frames(self, kind, d, seed, n):
        out = np.empty((n, d))
        k = {"static": 0, "dynamic": 1, "periodic": 2}[kind] if isinstance(kind, str) else kind
        self._check(self._f("stream_frames")(k, d, seed, n, _dp(out)))
        return out


@dataclass
class PipelineResult:
    seq: np.ndarray
    payload: np.ndarray | None
    report: dict
    decisions: np.ndarray | None


class _Engine:
    def __init__(self, o: Oracle, cfg: Cfg, cond, neg):
        self.o = o
        self.d = cfg.d_latent
        self.cfg = cfg
        self.h = C.c_void_p()
        self._cond = np.ascontiguousarray(cond, dtype=np.float64)
        self._neg = np.ascontiguousarray(neg, dtype=np.float64) if neg is not None else None
        o._check(o._f("engine_create")(C.byref(cfg), _dp(self._cond),
                                        _dp(self._neg) if self._neg is not None else None,
                                        C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.o._f("engine_destroy")(self.h)
            self.h = C.c_void_p()

    def ingest(self, seq, x0):
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        self.o._check(self.o._f("engine_ingest")(self.h, seq, _dp(x0)))

    def tick(self):
        es, it, et = C.c_int64(), C.c_int64(), C.c_int64()
        ca, ev = C.c_uint64(), C.c_uint64()
        out = np.empty(self.d)
        self.o._check(self.o._f("engine_tick")(self.h, C.byref(es), _dp(out), C.byref(it),
                                               C.byref(et), C.byref(ca), C.byref(ev)))
        emitted = None
        if es.value >= 0:
            emitted = dict(seq_id=es.value, x0_hat=out, ingest_tick=it.value, emit_tick=et.value)
        return dict(emitted=emitted, denoiser_calls=ca.value, element_evals=ev.value)

    def idle(self):
        return bool(self.o._f("engine_idle")(self.h))

    def ticks_completed(self):
        return self.o._f("engine_ticks")(self.h)

    def inflight_size(self):
        return self.o._f("engine_inflight")(self.h)

    def min_inflight_seq(self):
        v = self.o._f("engine_min_inflight_seq")(self.h)
        return None if v == 2**63 - 1 else v

    def step_indices(self):
        buf = (C.c_int * (self.cfg.n_steps + 1))()
        n = self.o._f("engine_step_indices")(self.h, buf)
        return list(buf[:n])

    def counters(self):
        a, b = C.c_uint64(), C.c_uint64()
        self.o._f("engine_counters")(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    def eps_cached(self, step):
        out = np.empty(self.d)
        self.o._f("engine_eps_cached")(self.h, step, _dp(out))
        return out


class _Ssf:
    def __init__(self, o: Oracle, eta, seed, max_skip):
        self.o = o
        self.h = C.c_void_p()
        if o.which == "orc":
            o._check(o._f("ssf_create")(eta, seed, max_skip, C.byref(self.h)))
        else:
            if max_skip > 0:
                raise ValueError("the reference has no max_skip (SURVEY §8c)")
            o._check(o._f("ssf_create")(eta, seed, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.o._f("ssf_destroy")(self.h)
            self.h = C.c_void_p()

    def gate(self, payload) -> int:
        p = np.ascontiguousarray(payload, dtype=np.float64)
        r = self.o._f("ssf_gate")(self.h, _dp(p), len(p))
        if r < 0:
            raise OracleError(-r, self.o._f("last_error")().decode())
        return r

    def counters(self):
        a, b = C.c_uint64(), C.c_uint64()
        self.o._f("ssf_counters")(self.h, C.byref(a), C.byref(b))
        return a.value, b.value


def load(which: str = "orc") -> Oracle:
    return Oracle(which)


def available(which: str) -> bool:
    return os.path.exists(PATHS[which])
