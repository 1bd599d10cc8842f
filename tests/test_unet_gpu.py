"""The batched device UNet (tcgen05 convs/GEMMs/attention, bf16 activations,
fp32 accumulation) against its PyTorch fp32 restatement (tests/unet_ref.py)
with the same weights.  Tolerance on eps (the UNet output, before the fp32
scheduler math): relative Frobenius error <= 3e-2 and per-row cosine >= 0.999,
the bf16-path bound for a ~70-layer network with bf16 activations."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def lib():
    from paper_2312_12491_b200 import _lib

    L = _lib.lib
    vp = C.c_void_p
    L.sdx_unet_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.c_uint64, C.c_int, C.POINTER(vp)]
    L.sdx_unet_forward.argtypes = [vp, vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), vp, vp]
    L.sdx_unet_param_count.argtypes = [vp, C.POINTER(C.c_int)]
    L.sdx_unet_param.argtypes = [vp, C.c_int, C.POINTER(C.c_char_p), C.POINTER(vp), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.sdx_unet_flops_per_row.argtypes = [vp, C.POINTER(C.c_double)]
    L.sdx_unet_profile.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_float),
                                   C.POINTER(C.c_int)]
    L.sdx_memcpy_d2d.argtypes = [vp, vp, C.c_int64]
    L.sdx_kernel_last_error.restype = C.c_char_p
    return L


@pytest.fixture(scope="module")
def unet(lib):
    taus = (C.c_int * 4)(999, 749, 499, 249)
    h = C.c_void_p()
    st = lib.sdx_unet_create(4, taus, 4, 1234, 0, C.byref(h))
    assert st == 0, lib.sdx_kernel_last_error()
    yield h
    lib.sdx_unet_destroy(h)


def run(lib, h, x, steps, prompts):
    R = x.shape[0]
    eps = torch.empty_like(x)
    st = lib.sdx_unet_forward(h, C.c_void_p(x.data_ptr()), R, (C.c_int * R)(*steps), (C.c_int * R)(*prompts),
                              C.c_void_p(eps.data_ptr()), None)
    assert st == 0, lib.sdx_kernel_last_error()
    return eps


def test_unet_matches_torch_fp32(lib, unet):
    from tests.unet_ref import export_params, unet_forward

    P = export_params(lib, unet)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(3, 64, 64, 4, device="cuda", generator=g)
    steps, prompts = [0, 2, 3], [0, 1, 0]
    eps = run(lib, unet, x, steps, prompts)
    taus = torch.tensor([[999, 749, 499, 249][s] for s in steps], device="cuda")
    with torch.no_grad():
        ref = unet_forward(P, x, taus, torch.tensor(prompts, device="cuda"))
    rel = float((eps - ref).norm() / ref.norm())
    cos = torch.nn.functional.cosine_similarity(eps.flatten(1), ref.flatten(1)).min().item()
    print(f"unet eps rel err {rel:.3e}, min row cosine {cos:.6f}, |ref| {ref.abs().max().item():.3f}")
    assert torch.isfinite(eps).all()
    assert rel <= 3e-2 and cos >= 0.999


def test_unet_rows_are_independent(lib, unet):
    # the device-decided row count: rows past it do no work, live rows do not
    # depend on how many rows the batch holds
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(4, 64, 64, 4, device="cuda", generator=g)
    full = run(lib, unet, x, [0, 1, 2, 3], [0, 0, 1, 1])
    part = run(lib, unet, x[:2].contiguous(), [0, 1], [0, 0])
    assert torch.equal(full[:2], part)


def test_unet_flops_and_profile(lib, unet):
    f = C.c_double()
    assert lib.sdx_unet_flops_per_row(unet, C.byref(f)) == 0
    # SD-2.1 topology at 64x64 latent: ~0.8 TFLOP per row
    assert 7.0e11 < f.value < 9.0e11, f.value
    kinds = (C.c_char_p * 1024)()
    ms = (C.c_float * 1024)()
    n = C.c_int()
    assert lib.sdx_unet_profile(unet, 4, 1024, kinds, ms, C.byref(n)) == 0
    tot = {}
    for i in range(n.value):
        tot[kinds[i].decode()] = tot.get(kinds[i].decode(), 0.0) + ms[i]
    print("unet op times (ms, 4 rows):", {k: round(v, 3) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])})
    print("total ms", sum(tot.values()), "TFLOP/s", 4 * f.value / (sum(tot.values()) * 1e-3) / 1e12)
