"""ctypes binding of the C-ABI (include/stagger_b200.h) of libstagger_b200.so.

The library is built in-tree (paper_2312_12491_b200/build.py or
__graft_entry__.build()).  There is no fallback: if the shared object is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libstagger_b200.so")

SDX_OK, SDX_INVALID_ARGUMENT, SDX_LOGIC_ERROR, SDX_RUNTIME_ERROR, SDX_CUDA_ERROR, SDX_UNSUPPORTED = range(6)
GUIDANCE = {"none": 0, "cfg": 1, "self_negative": 2, "onetime_negative": 3}
LCM = {"exact": 0, "boundary_approx": 1}
BACKEND = {"analytic": 0, "unet": 2}
CODEC = {"identity": 0, "taesd": 2}


class sdx_config(C.Structure):
    _fields_ = [
        ("n_steps", C.c_int), ("guidance_mode", C.c_int), ("gamma", C.c_double), ("delta", C.c_double),
        ("ssf_enabled", C.c_int), ("eta", C.c_double), ("seed", C.c_uint64),
        ("cross_frame_attention", C.c_int), ("d_latent", C.c_int), ("t_grid", C.c_int),
        ("entry_strength", C.c_double), ("backend", C.c_int), ("data_variance", C.c_double),
        ("lcm_mode", C.c_int), ("codec", C.c_int), ("queue_capacity", C.c_int),
    ]


class sdx_step(C.Structure):
    _fields_ = [("tau", C.c_int), ("alpha", C.c_double), ("beta", C.c_double)]


class sdx_tick_result(C.Structure):
    _fields_ = [("emitted_seq", C.c_int64), ("ingest_tick", C.c_int64), ("emit_tick", C.c_int64),
                ("denoiser_calls", C.c_uint64), ("element_evals", C.c_uint64)]


class sdx_pipeline_config(C.Structure):
    _fields_ = [("engine", sdx_config), ("n_streams", C.c_int), ("frame_bytes", C.c_int64),
                ("max_skip", C.c_int), ("ring_depth", C.c_int), ("graph", C.c_int)]


class sdx_trace_entry(C.Structure):
    _fields_ = [("tick", C.c_int64), ("ingested", C.c_int64), ("emitted", C.c_int64), ("calls", C.c_uint64),
                ("element_evals", C.c_uint64), ("elapsed_ns", C.c_int64)]


class sdx_report(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "frames_in", "frames_out", "duplicates", "stale_skips", "input_drops", "output_drops", "ticks",
        "denoiser_calls", "element_evals", "ssf_examined", "ssf_skipped")] + [
        ("skip_rate", C.c_double), ("latency_ticks_mean", C.c_double), ("latency_ticks_min", C.c_int64),
        ("latency_ticks_max", C.c_int64), ("mean_frame_time_ms", C.c_double), ("throughput_fps", C.c_double),
        ("wall_ms", C.c_double), ("incomplete", C.c_int)]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python {HERE}/build.py` "
                      "(the product has no CPU fallback)")
lib = C.CDLL(LIB_PATH)

P = C.c_void_p
D = C.POINTER(C.c_double)
_sig = {
    "sdx_last_error": (C.c_char_p, []),
    "sdx_abi_version": (C.c_int, []),
    "sdx_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "sdx_engine_create": (C.c_int, [C.POINTER(sdx_config), C.POINTER(sdx_step), C.c_int, D, D, C.c_int,
                                    C.POINTER(P)]),
    "sdx_engine_destroy": (C.c_int, [P]),
    "sdx_engine_ingest": (C.c_int, [P, C.c_int64, D, D]),
    "sdx_engine_tick": (C.c_int, [P, C.POINTER(sdx_tick_result), D]),
    "sdx_engine_ticks_completed": (C.c_int, [P, C.POINTER(C.c_int64)]),
    "sdx_engine_inflight": (C.c_int, [P, C.POINTER(C.c_int)]),
    "sdx_engine_step_indices": (C.c_int, [P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sdx_engine_min_inflight_seq": (C.c_int, [P, C.POINTER(C.c_int64)]),
    "sdx_engine_counters": (C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "sdx_engine_reset_counters": (C.c_int, [P]),
    "sdx_engine_last_tick_ms": (C.c_int, [P, C.POINTER(C.c_float)]),
    "sdx_ssf_create": (C.c_int, [C.c_double, C.c_uint64, C.c_int, C.c_int64, C.c_int, C.POINTER(P)]),
    "sdx_ssf_destroy": (C.c_int, [P]),
    "sdx_ssf_gate": (C.c_int, [P, C.c_void_p, C.c_int, C.POINTER(C.c_int), D]),
    "sdx_ssf_counters": (C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "sdx_pipeline_create": (C.c_int, [C.POINTER(sdx_pipeline_config), C.POINTER(sdx_step), D, D, D, C.c_int,
                                      C.POINTER(P)]),
    "sdx_pipeline_destroy": (C.c_int, [P]),
    "sdx_pipeline_push": (C.c_int, [P, C.c_void_p]),
    "sdx_pipeline_push_seq": (C.c_int, [P, C.c_void_p, C.c_void_p]),
    "sdx_pipeline_tick": (C.c_int, [P, C.POINTER(C.c_int)]),
    "sdx_pipeline_idle": (C.c_int, [P, C.POINTER(C.c_int)]),
    "sdx_pipeline_finish": (C.c_int, [P]),
    "sdx_pipeline_pop": (C.c_int, [P, C.c_int, C.POINTER(C.c_int64), C.c_void_p, C.POINTER(C.c_int)]),
    "sdx_pipeline_report": (C.c_int, [P, C.c_int, C.POINTER(sdx_report)]),
    "sdx_pipeline_decisions": (C.c_int, [P, C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int)]),
    "sdx_pipeline_trace": (C.c_int, [P, C.c_int, C.POINTER(sdx_trace_entry), C.c_int, C.POINTER(C.c_int)]),
    "sdx_pipeline_sync": (C.c_int, [P]),
    "sdx_pipeline_error_message": (C.c_char_p, [P, C.c_int]),
    "sdx_pipeline_device_time_ms": (C.c_int, [P, C.POINTER(C.c_float)]),
    "sdx_pipeline_reset_timer": (C.c_int, [P]),
    "sdx_pipeline_upload_resident": (C.c_int, [P, C.c_void_p, C.c_int]),
    "sdx_pipeline_push_resident": (C.c_int, [P, C.c_int]),
    "sdx_pipeline_set_profile": (C.c_int, [P, C.c_int]),
    "sdx_pipeline_stage_times": (C.c_int, [P, D, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "sdx_pipeline_flops": (C.c_int, [P, D, D]),
    "sdx_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "sdx_build_schedule": (C.c_int, [C.c_int, C.c_int, C.c_double, C.POINTER(sdx_step)]),
    "sdx_sample_gaussian": (C.c_int, [C.c_uint64, C.c_int64, D]),
    "sdx_build_noise_cache": (C.c_int, [C.c_uint64, C.c_int, C.c_int64, D]),
    "sdx_precompute_error": (C.c_char_p, []),
    "sdx_profiler_start": (C.c_int, []),
    "sdx_profiler_stop": (C.c_int, []),
    "sdx_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "sdx_host_free": (C.c_int, [C.c_void_p]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = sorted(_sig)
