"""GPU parity of the device-decided pipeline (sdx_pipeline_*) against the
oracle's deterministic run_pipeline (pipeline.cpp:152-214): sink order and
duplicate placement bit-exact, SSF decisions bit-exact, report counters
identical, payloads within 1e-3 (fp32 latents).  Mirrors test_runtime.cpp."""
import numpy as np
import pytest

from oracle.oracle import make_cfg

pytestmark = pytest.mark.gpu
TOL = 1e-3
INT_KEYS = ["frames_in", "frames_out", "duplicates", "stale_skips", "input_drops", "output_drops", "ticks",
            "denoiser_calls", "element_evals", "ssf_examined", "ssf_skipped", "latency_ticks_min",
            "latency_ticks_max"]


def u8_stream(kind, D, seed, n):
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 256, D, dtype=np.uint8)
    out = []
    for i in range(n):
        if kind == "static":
            f = base
        elif kind == "dynamic":
            f = rng.integers(0, 256, D, dtype=np.uint8)
        else:  # near-static with cuts: sims straddle 0.98
            if i % 23 == 22:
                base = rng.integers(0, 256, D, dtype=np.uint8)
            f = base.copy()
            k = int(rng.integers(0, D // 30))
            idx = rng.integers(0, D, k)
            f[idx] = rng.integers(0, 256, k, dtype=np.uint8)
        out.append(f)
    return np.stack(out)


def compare(sg, orc, frames, n, mode="none", ssf=True, seed=3, max_skip=0, lcm="exact", xfa=False):
    D = frames.shape[1]
    neg = orc.gaussian(orc.derive_seed(seed, 5), D) if mode in ("cfg", "onetime_negative") else None
    ocfg = make_cfg(n_steps=n, guidance_mode=mode, ssf_enabled=ssf, seed=seed, d_latent=D, lcm_mode=lcm,
                    cross_frame_attention=xfa)
    want = orc.run_pipeline(ocfg, frames.astype(np.float64), neg=neg, max_skip=max_skip)
    cfg = sg.EngineConfig(n_steps=n, guidance_mode=mode, ssf_enabled=ssf, seed=seed, d_latent=D,
                          negative_condition=neg, lcm_mode=lcm, cross_frame_attention=xfa)
    sink, rep = sg.run_pipeline(cfg, frames, max_skip=max_skip)
    assert [s for s, _ in sink] == want.seq.tolist()
    worst = max((float(np.max(np.abs(p.astype(np.float64) - w))) for (_, p), w in zip(sink, want.payload)),
                default=0.0)
    assert worst <= TOL, worst
    for k in INT_KEYS:
        assert rep[k] == want.report[k], (k, rep[k], want.report[k])
    assert rep["incomplete"] is False
    for k in ("skip_rate", "latency_ticks_mean", "mean_frame_time_ms", "throughput_fps", "wall_ms"):
        assert rep[k] == pytest.approx(want.report[k], rel=1e-12)
    return want, sink, rep


@pytest.mark.parametrize("kind", ["static", "dynamic", "periodic"])
@pytest.mark.parametrize("n", [1, 4])
def test_pipeline_matches_oracle(sg, orc, kind, n):
    frames = u8_stream(kind, 1024, 10 + n, 120)
    compare(sg, orc, frames, n)


@pytest.mark.parametrize("mode", ["none", "cfg", "self_negative", "onetime_negative"])
def test_pipeline_modes(sg, orc, mode):
    frames = u8_stream("periodic", 2048, 4, 80)
    compare(sg, orc, frames, 3, mode=mode)


def test_pipeline_static_scene_duplicates(sg, orc):
    # test_runtime.cpp:169-188 shape: one processed frame, duplicates for the rest
    frames = u8_stream("static", 512, 1, 20)
    want, sink, rep = compare(sg, orc, frames, 4)
    assert rep["ssf_skipped"] == 19 and rep["duplicates"] == 19 and rep["element_evals"] == 4


def test_pipeline_ssf_off_equals_on_for_dynamic(sg, orc):
    # test_runtime.cpp:190-211
    frames = u8_stream("dynamic", 1024, 2, 60)
    _, a, _ = compare(sg, orc, frames, 3, ssf=False)
    _, b, rep = compare(sg, orc, frames, 3, ssf=True)
    assert rep["ssf_skipped"] == 0
    assert [s for s, _ in a] == [s for s, _ in b]
    for (_, x), (_, y) in zip(a, b):
        assert np.array_equal(x, y)


def test_pipeline_max_skip(sg, orc):
    frames = u8_stream("static", 4096, 3, 60)
    want, _, rep = compare(sg, orc, frames, 2, max_skip=10)
    assert rep["ssf_skipped"] < 59


def test_pipeline_latent_16384(sg, orc):
    # the 4x64x64 latent size, near-static stream
    frames = u8_stream("periodic", 16384, 5, 40)
    compare(sg, orc, frames, 4, mode="self_negative")


def test_multistream_equals_independent_streams(sg, orc):
    # cfg4 shape: S streams batched into one tick == S independent runs with seed base+s
    S, D, n, N = 8, 1024, 1, 50
    streams = [u8_stream("periodic", D, 100 + s, N) for s in range(S)]
    cfg = sg.EngineConfig(n_steps=n, guidance_mode="self_negative", ssf_enabled=True, seed=40, d_latent=D)
    p = sg.Pipeline(cfg, S, D)
    sinks = [[] for _ in range(S)]
    for i in range(N):
        p.push(np.stack([streams[s][i] for s in range(S)]))
        for s in range(S):
            sinks[s].extend(p.pop_all(s))
    p.finish()
    for s in range(S):
        sinks[s].extend(p.pop_all(s))
        want = orc.run_pipeline(make_cfg(n_steps=n, guidance_mode="self_negative", ssf_enabled=True, seed=40 + s,
                                         d_latent=D), streams[s].astype(np.float64))
        assert [q for q, _ in sinks[s]] == want.seq.tolist()
        assert p.decisions(s).tolist() == want.decisions.tolist()
        for (_, x), w in zip(sinks[s], want.payload):
            assert np.max(np.abs(x - w)) <= TOL
        rep = p.report(s)
        for k in INT_KEYS:
            assert rep[k] == want.report[k], (s, k)
    p.close()


def test_pipeline_failure_marks_incomplete(sg):
    # test_runtime.cpp:303-316 analogue: a frame of the wrong width is rejected
    cfg = sg.EngineConfig(n_steps=2, d_latent=8)
    p = sg.Pipeline(cfg, 1, 8)
    p.push(np.ones(8, dtype=np.uint8))
    with pytest.raises(sg.InvalidArgument):
        p.push(np.ones(3, dtype=np.uint8))
    p.close()


@pytest.mark.parametrize("n,mode", [(2, "none"), (4, "cfg"), (3, "onetime_negative")])
def test_pipeline_tick_trace(sg, orc, n, mode):
    # engine.cpp:181-192 / pipeline.cpp:135-148: one TickLogEntry per tick, ticks 1..T, each
    # emission the oldest in-flight frame, per-tick denoiser counters summing to the report's
    D = 512
    frames = u8_stream("periodic", D, 17, 40)
    neg = orc.gaussian(orc.derive_seed(3, 5), D) if mode in ("cfg", "onetime_negative") else None
    cfg = sg.EngineConfig(n_steps=n, guidance_mode=mode, ssf_enabled=True, seed=3, d_latent=D,
                          negative_condition=neg)
    p = sg.Pipeline(cfg, n_streams=1, frame_bytes=D)
    for f in frames:
        p.push(f[None])
    p.finish()
    p.sync()
    rep = p.report(0)
    tr = p.trace(0)
    p.close()
    assert len(tr) == rep["ticks"] and [e["tick"] for e in tr] == list(range(1, len(tr) + 1))
    assert sum(e["calls"] for e in tr) == rep["denoiser_calls"]
    assert sum(e["element_evals"] for e in tr) == rep["element_evals"]
    ingested = [e["ingested"] for e in tr if e["ingested"] is not None]
    emitted = [e["emitted"] for e in tr if e["emitted"] is not None]
    assert ingested == sorted(ingested) and emitted == sorted(emitted)
    assert emitted == ingested  # every processed frame is emitted once, in order
    for e in tr:  # emission happens n ticks after ingestion (latency n)
        if e["emitted"] is not None:
            t_in = next(x["tick"] for x in tr if x["ingested"] == e["emitted"])
            assert e["tick"] - t_in == n - 1


@pytest.mark.parametrize("mode", ["none", "self_negative", "onetime_negative"])
@pytest.mark.parametrize("n", [2, 4])
def test_pipeline_cross_frame_attention(sg, orc, mode, n):
    # test_stream_batch.cpp:284-308 (cross-frame attention keeps latency n and ordering) and the
    # device pipeline's sink / report / payloads against the oracle's run_pipeline with it on
    frames = u8_stream("periodic", 256, 51 + n, 40)
    want, sink, rep = compare(sg, orc, frames, n, mode=mode, xfa=True)
    assert rep["latency_ticks_min"] == rep["latency_ticks_max"] == n


def test_pipeline_source_seq_ids(sg, orc):
    # the sink, duplicates and trace carry the source's Frame::seq_id (pipeline.cpp:176):
    # sparse ids map one to one onto the frame-index run
    D, n = 1024, 3
    frames = u8_stream("periodic", D, 61, 70)
    ids = [500 + 7 * i for i in range(len(frames))]
    cfg = sg.EngineConfig(n_steps=n, ssf_enabled=True, seed=9, d_latent=D)
    base, rep0 = sg.run_pipeline(cfg, frames)
    sink, rep = sg.run_pipeline(cfg, frames, seq_ids=ids)
    assert rep["duplicates"] == rep0["duplicates"] > 0
    assert [s for s, _ in sink] == [ids[s] for s, _ in base]
    for (_, a), (_, b) in zip(sink, base):
        assert np.array_equal(a, b)
    # trace ids are source ids as well
    p = sg.Pipeline(cfg, 1, D)
    for i, f in enumerate(frames):
        p.push(f[None], [ids[i]])
    p.finish()
    ingested = {e["ingested"] for e in p.trace(0) if e["ingested"] is not None}
    p.close()
    assert ingested <= set(ids) and len(ingested) == len(frames) - rep["ssf_skipped"]


def test_pipeline_seq_ids_must_increase(sg):
    # engine.cpp:59-60: an ingested frame whose id does not increase fails the stream
    D = 256
    cfg = sg.EngineConfig(n_steps=2, d_latent=D)
    frames = u8_stream("dynamic", D, 3, 6)
    sink, rep = sg.run_pipeline(cfg, frames, seq_ids=[0, 1, 2, 3, 2, 5])
    assert rep["incomplete"] and "strictly increase" in rep["error"]


def test_pipeline_tick_without_input(sg, orc):
    # pipeline.cpp:235-245: the live loop ticks a non-idle engine when no input waits; the
    # frames in flight complete with latency n and the same payloads as a flushed run
    D, n = 512, 4
    frames = u8_stream("dynamic", D, 8, 3)
    cfg = sg.EngineConfig(n_steps=n, seed=4, d_latent=D)
    want, _ = sg.run_pipeline(cfg, frames)
    p = sg.Pipeline(cfg, 1, D)
    for f in frames:
        p.push(f[None])
    ran = 0
    while p.tick():
        ran += 1
        assert ran < 50
    assert p.idle()
    got = p.pop_all(0)
    rep = p.report(0)
    p.close()
    assert ran >= n - 1
    assert [s for s, _ in got] == [s for s, _ in want]
    for (_, a), (_, b) in zip(got, want):
        assert np.array_equal(a, b)
    assert rep["latency_ticks_min"] == rep["latency_ticks_max"] == n


def test_resident_no_copy_counts_duplicates(sg, orc):
    # benchmark mode without output copies: skipped frames still become duplicates once
    # a frame was emitted (has-output flag independent of the payload copy)
    D = 1024
    frames = u8_stream("static", D, 2, 4)
    cfg = sg.EngineConfig(n_steps=1, ssf_enabled=True, seed=3, d_latent=D)
    want = orc.run_pipeline(make_cfg(n_steps=1, ssf_enabled=True, seed=3, d_latent=D),
                            np.concatenate([frames] * 3).astype(np.float64))
    p = sg.Pipeline(cfg, 1, D, ring_depth=4)
    p.upload_resident(frames)
    for _ in range(12):
        p.push_resident(copy_outputs=False)
    p.finish()
    p.sync()
    rep = p.report(0)
    p.close()
    for k in ("duplicates", "stale_skips", "frames_out", "ssf_skipped"):
        assert rep[k] == want.report[k], (k, rep[k], want.report[k])
