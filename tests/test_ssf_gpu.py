"""GPU parity of the device SSF gate (sdx_ssf_*): decisions and cosines are
bit-exact against the oracle's SsfState on u8 frames (exact integer sums,
IEEE fp64 tail, device MT19937-64).  Mirrors test_ssf.cpp and SURVEY §8d cfg3.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "engine_golden.json")


def near_static_stream(rng, D, nframes, base=None, cut_every=0, k_max=None):
    """Base image plus sparse +-k perturbations (sims straddle eta) and
    occasional scene cuts."""
    base = rng.integers(0, 256, D, dtype=np.uint8) if base is None else base
    k_max = k_max or max(1, D // 40)
    for i in range(nframes):
        if cut_every and i % cut_every == cut_every - 1:
            base = rng.integers(0, 256, D, dtype=np.uint8)
        f = base.copy()
        k = int(rng.integers(0, k_max))
        idx = rng.integers(0, D, k)
        f[idx] = rng.integers(0, 256, k, dtype=np.uint8)
        yield f


def oracle_decisions(orc, frames, eta, seed, max_skip=0):
    g = orc.ssf(eta, seed, max_skip)
    dec = [g.gate(f.astype(np.float64)) for f in frames]
    return np.array(dec, dtype=np.int32)


def test_golden_ssf_decisions(sg):
    g = json.load(open(GOLDEN))["ssf"]
    frames = np.array(g["frames"], dtype=np.uint8)
    s = sg.SsfState(g["eta"], g["seed"], frames.shape[1])
    dec = s.gate_many(frames)
    assert dec.tolist() == g["decisions"]


@pytest.mark.parametrize("max_skip", [0, 10])
def test_decisions_bitexact_10k(sg, orc, max_skip):
    # >= 1e4 frames, sims straddling eta = 0.98, scene cuts
    rng = np.random.default_rng(7)
    D = 3 * 32 * 32
    frames = np.stack(list(near_static_stream(rng, D, 10000, cut_every=997, k_max=60)))
    seed = orc.derive_seed(11, 2)
    want = oracle_decisions(orc, frames, 0.98, seed, max_skip)
    s = sg.SsfState(0.98, seed, D, max_skip=max_skip)
    got, sims = s.gate_many(frames, with_sims=True)
    assert 0.05 < want.mean() < 0.95  # the stream exercises both outcomes
    np.testing.assert_array_equal(got, want)
    # cosines equal the oracle bit for bit (first frame: NaN marker)
    ref = frames[0].astype(np.float64)
    for i in range(1, 200):
        if want[i - 1] == 0:
            ref = frames[i - 1].astype(np.float64)
        assert sims[i] == orc.cosine(frames[i].astype(np.float64), ref)
    assert s.counters() == (10000, int(want.sum()))


def test_decisions_bitexact_512(sg, orc):
    # full 3x512x512 frames
    rng = np.random.default_rng(3)
    D = 3 * 512 * 512
    frames = list(near_static_stream(rng, D, 48, cut_every=16, k_max=20000))
    seed = orc.derive_seed(5, 2)
    want = oracle_decisions(orc, frames, 0.98, seed)
    got = sg.SsfState(0.98, seed, D).gate_many(np.stack(frames))
    np.testing.assert_array_equal(got, want)


def test_static_stream_skips_all_but_first(sg):
    # test_ssf.cpp:97-104
    f = np.arange(1000, dtype=np.uint8)[None].repeat(1001, 0)
    s = sg.SsfState(0.98, 2, 1000)
    dec = s.gate_many(f)
    assert dec[0] == 0 and dec[1:].all()
    assert s.counters() == (1001, 1000)


def test_never_skips_below_threshold(sg, orc):
    # test_ssf.cpp:106-115: independent random frames sit far below eta
    rng = np.random.default_rng(1)
    frames = rng.integers(0, 256, (300, 4096), dtype=np.uint8)
    dec = sg.SsfState(0.9, 3, 4096).gate_many(frames)
    # uniform u8 frames have cosine ~0.75 < 0.9
    assert not dec.any()


def test_zero_norm_frame_fails_open(sg):
    # cosine of a zero frame is 0 (ssf.cpp:17) -> never skipped at eta >= 0
    frames = np.zeros((20, 512), dtype=np.uint8)
    frames[0] = 7
    dec = sg.SsfState(0.5, 4, 512).gate_many(frames)
    assert not dec.any()


def test_odd_frame_size_tail(sg, orc):
    # D not a multiple of 16 exercises the scalar tail
    rng = np.random.default_rng(9)
    D = 1001
    frames = list(near_static_stream(rng, D, 500, cut_every=50, k_max=40))
    seed = 1234
    np.testing.assert_array_equal(sg.SsfState(0.98, seed, D).gate_many(np.stack(frames)),
                                  oracle_decisions(orc, frames, 0.98, seed))
