"""GPU parity of the device StreamBatchEngine (C-ABI sdx_engine_*) against
the CPU oracle (oracle/stagger_oracle.c, itself pinned bit-for-bit to the
reference build).  Mirrors test_stream_batch.cpp.

Tolerance: the device path stores latents in fp32 and computes in fp64, so
emitted x0_hat must match the fp64 oracle to max-abs <= 1e-3 (north_star's
fp32-path bound); observed deviations are ~1e-6.  Tick/latency/ordering
observables must be identical.
"""
import numpy as np
import pytest

from oracle.oracle import make_cfg

pytestmark = pytest.mark.gpu
MODES = ["none", "cfg", "self_negative", "onetime_negative"]
TOL = 1e-3


def pair(sg, orc, n, mode, d, lcm="exact", seed=0, entry=1.0, xfa=False):
    cond = orc.gaussian(orc.derive_seed(seed, 4), d)
    neg = orc.gaussian(orc.derive_seed(seed, 5), d)
    use_neg = neg if mode in ("cfg", "onetime_negative") else None
    ocfg = make_cfg(n_steps=n, guidance_mode=mode, d_latent=d, lcm_mode=lcm, seed=seed, entry_strength=entry,
                    cross_frame_attention=xfa)
    eo = orc.engine(ocfg, cond, use_neg)
    cfg = sg.EngineConfig(n_steps=n, guidance_mode=mode, d_latent=d, lcm_mode=lcm, seed=seed,
                          entry_strength=entry, negative_condition=use_neg, cross_frame_attention=xfa)
    ed = sg.StreamBatchEngine(cfg)
    return ed, eo, cond


def drive(ed, eo, cond, xs, bubble_every=0):
    """Feed both engines; returns max deviation over emitted frames."""
    worst = 0.0
    emitted = 0
    for seq, x in enumerate(xs):
        if not (bubble_every and seq % bubble_every == bubble_every - 1):
            ed.ingest(seq, x, cond)
            eo.ingest(seq, x)
        if eo.idle():
            assert ed.idle()
            continue
        a, b = ed.tick(), eo.tick()
        assert a.element_evals == b["element_evals"] and a.denoiser_calls == 1
        assert (a.emitted is None) == (b["emitted"] is None)
        if a.emitted:
            emitted += 1
            assert a.emitted.seq_id == b["emitted"]["seq_id"]
            assert (a.emitted.ingest_tick, a.emitted.emit_tick) == (b["emitted"]["ingest_tick"],
                                                                    b["emitted"]["emit_tick"])
            worst = max(worst, float(np.max(np.abs(a.emitted.x0_hat - b["emitted"]["x0_hat"]))))
        assert ed.step_indices() == eo.step_indices()
        assert ed.min_inflight_seq() == eo.min_inflight_seq()
        assert ed.ticks_completed() == eo.ticks_completed()
    while not eo.idle():
        a, b = ed.tick(), eo.tick()
        if a.emitted:
            emitted += 1
            assert a.emitted.seq_id == b["emitted"]["seq_id"]
            worst = max(worst, float(np.max(np.abs(a.emitted.x0_hat - b["emitted"]["x0_hat"]))))
    assert ed.idle()
    assert ed.counters() == eo.counters()
    return worst, emitted


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n", [1, 2, 4, 10])
def test_engine_matches_oracle_small(sg, orc, n, mode):
    # test_stream_batch.cpp:250-282 at d = 8, both LCM modes, with bubbles
    for lcm in ("exact", "boundary_approx"):
        ed, eo, cond = pair(sg, orc, n, mode, 8, lcm)
        rng = np.random.default_rng(13)
        xs = [rng.standard_normal(8) for _ in range(25)]
        worst, emitted = drive(ed, eo, cond, xs, bubble_every=7)
        assert emitted > 0 and worst <= TOL, worst
        ed.close()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n", [1, 4])
def test_engine_matches_oracle_latent_16384(sg, orc, n, mode):
    # the 4x64x64 latent of the B200 build
    d = 16384
    ed, eo, cond = pair(sg, orc, n, mode, d, entry=1.0, seed=1)
    rng = np.random.default_rng(2)
    xs = [rng.standard_normal(d) for _ in range(2 * n + 3)]
    worst, emitted = drive(ed, eo, cond, xs)
    assert emitted == len(xs) and worst <= TOL, worst


def test_txt2img_zero_latent(sg, orc):
    # cfg0: txt2img emulated as ingest(seq, zeros)
    d = 16384
    for mode in ("none", "self_negative"):
        ed, eo, cond = pair(sg, orc, 1, mode, d)
        worst, emitted = drive(ed, eo, cond, [np.zeros(d)])
        assert emitted == 1 and worst <= TOL


def test_latency_and_staggering(sg, orc):
    # test_stream_batch.cpp:99-159
    n = 4
    ed, eo, cond = pair(sg, orc, n, "none", 8)
    rng = np.random.default_rng(5)
    for t in range(n - 1):
        ed.ingest(t, rng.standard_normal(8), cond)
        assert ed.step_indices() == list(range(t + 1))
        assert ed.tick().emitted is None
    for t in range(n - 1, 30):
        ed.ingest(t, rng.standard_normal(8), cond)
        assert ed.step_indices() == list(range(n))
        r = ed.tick()
        assert r.emitted is not None and r.denoiser_calls == 1
        assert r.emitted.emit_tick - r.emitted.ingest_tick == n


def test_error_contract(sg, orc):
    ed, _, cond = pair(sg, orc, 4, "none", 8)
    with pytest.raises(sg.LogicError):  # tick on an empty engine
        ed.tick()
    ed.ingest(5, np.ones(8), cond)
    with pytest.raises(sg.LogicError):  # double ingest without a tick
        ed.ingest(6, np.ones(8), cond)
    ed.tick()
    with pytest.raises(sg.InvalidArgument):  # seq ids must strictly increase
        ed.ingest(5, np.ones(8), cond)
    with pytest.raises(sg.InvalidArgument):  # non-finite latent
        ed.ingest(9, np.full(8, np.nan), cond)
    with pytest.raises(sg.InvalidArgument):  # wrong width
        ed.ingest(9, np.ones(3), cond)


def test_nonfinite_emission_raises(sg, orc):
    # engine.cpp:166-168: non-finite latent at emission -> runtime_error.  gamma = inf
    # passes validate_config (gamma >= 0) and makes the CFG combine non-finite in both
    # the fp64 reference and the device path.
    from oracle.oracle import OracleError

    d = 8
    neg = np.linspace(-1, 1, d)
    ocfg = make_cfg(n_steps=1, guidance_mode="cfg", gamma=float("inf"), d_latent=d)
    eo = orc.engine(ocfg, np.zeros(d), neg)
    eo.ingest(0, np.ones(d))
    with pytest.raises(OracleError) as ei:
        eo.tick()
    assert ei.value.code == 3
    cfg = sg.EngineConfig(n_steps=1, guidance_mode="cfg", gamma=float("inf"), d_latent=d, negative_condition=neg)
    ed = sg.StreamBatchEngine(cfg)
    ed.ingest(0, np.ones(d), np.zeros(d))
    with pytest.raises(sg.StaggerRuntimeError):
        ed.tick()


def test_bubbles_advance_partial_batch(sg, orc):
    # test_stream_batch.cpp:187-202
    n = 4
    ed, eo, cond = pair(sg, orc, n, "none", 8)
    ed.ingest(0, np.ones(8), cond)
    for _ in range(n - 1):
        assert ed.tick().emitted is None
    r = ed.tick()
    assert r.emitted is not None and r.emitted.emit_tick - r.emitted.ingest_tick == n
    assert ed.idle()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("d,scale", [(8, 1.0), (64, 0.3), (16384, 0.02)])
def test_engine_cross_frame_attention_matches_oracle(sg, orc, n, mode, d, scale):
    # engine.cpp:139-149 + attention.cpp:12-95 on the device (three launches per tick) vs the C
    # restatement (bit-exact with the reference build): emissions within the fp32 bound, all
    # tick / ordering observables identical; `scale` keeps the attention weights mixed
    ed, eo, cond = pair(sg, orc, n, mode, d, xfa=True)
    rng = np.random.default_rng(29 + n)
    xs = [scale * rng.standard_normal(d) for _ in range(3 * n + 8)]
    worst, emitted = drive(ed, eo, cond, xs, bubble_every=5)
    assert emitted > 0 and worst <= TOL, worst
    ed.close()
