"""The full B200 path (device SSF -> TAESD encode -> batched UNet -> fused
R-CFG/LCM step -> TAESD decode) against the reference pipeline's observable
contract: the skip/run decisions, the sink order with duplicates at their
sequence position and the report counters are functions of the frames and
n only, so they must equal the oracle's run_pipeline on the same u8 frames
bit for bit, whatever the denoiser."""
import numpy as np
import pytest

from oracle.oracle import make_cfg

pytestmark = pytest.mark.gpu
D = 3 * 512 * 512
INT_KEYS = ["frames_in", "frames_out", "duplicates", "stale_skips", "ticks", "denoiser_calls", "element_evals",
            "ssf_examined", "ssf_skipped", "latency_ticks_min", "latency_ticks_max"]


def stream(seed, n, cut_every=9):
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 256, D, dtype=np.uint8)
    out = []
    for i in range(n):
        if i % cut_every == cut_every - 1:
            base = rng.integers(0, 256, D, dtype=np.uint8)
        f = base.copy()
        k = int(rng.integers(0, 30000))
        idx = rng.integers(0, D, k)
        f[idx] = rng.integers(0, 256, k, dtype=np.uint8)
        out.append(f)
    return np.stack(out)


@pytest.mark.parametrize("n,guidance,S", [(4, "none", 1), (1, "self_negative", 3), (2, "onetime_negative", 2),
                                          (2, "cfg", 2)])
def test_unet_taesd_pipeline_contract(sg, orc, n, guidance, S):
    N = 24
    streams = [stream(50 + s, N) for s in range(S)]
    neg = sg.sample_gaussian(sg.derive_seed(0, 5), 4 * 64 * 64) if guidance in ("cfg", "onetime_negative") else None
    cfg = sg.EngineConfig(n_steps=n, guidance_mode=guidance, ssf_enabled=True, eta=0.98, seed=10, d_latent=4 * 64 * 64,
                          backend="unet", codec="taesd", negative_condition=neg)
    p = sg.Pipeline(cfg, S, D)
    sinks = [[] for _ in range(S)]
    for i in range(N):
        p.push(np.stack([streams[s][i] for s in range(S)]))
        for s in range(S):
            sinks[s].extend(p.pop_all(s))
    p.finish()
    for s in range(S):
        sinks[s].extend(p.pop_all(s))
        onegd = orc.gaussian(orc.derive_seed(10 + s, 5), D) if guidance in ("cfg", "onetime_negative") else None
        want = orc.run_pipeline(make_cfg(n_steps=n, guidance_mode=guidance, ssf_enabled=True, seed=10 + s, d_latent=D),
                                streams[s].astype(np.float64), neg=onegd, want_payload=False)
        assert p.decisions(s).tolist() == want.decisions.tolist()
        assert [q for q, _ in sinks[s]] == want.seq.tolist()
        rep = p.report(s)
        assert not rep["incomplete"], rep["error"]
        for k in INT_KEYS:
            assert rep[k] == want.report[k], (s, k, rep[k], want.report[k])
        # payloads are decoded u8 frames; duplicates replay the last emitted output
        last = None
        dec = p.decisions(s)
        for (seq, pay) in sinks[s]:
            assert pay.dtype == np.uint8 and pay.size == D
            if dec[seq] == 1 and last is not None:
                assert np.array_equal(pay, last)
            else:
                last = pay
        assert 0.05 < dec.mean() < 0.95
    p.close()


def test_unet_taesd_outputs_vary_with_input(sg):
    cfg = sg.EngineConfig(n_steps=1, guidance_mode="self_negative", ssf_enabled=False, seed=3, d_latent=4 * 64 * 64,
                          backend="unet", codec="taesd")
    p = sg.Pipeline(cfg, 2, D)
    fr = stream(1, 2, cut_every=1)
    p.push(fr)
    p.finish()
    a, b = p.pop_all(0), p.pop_all(1)
    assert len(a) == 1 and len(b) == 1
    assert not np.array_equal(a[0][1], b[0][1])
    assert a[0][1].std() > 0
    p.close()
