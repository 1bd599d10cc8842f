"""Numerics of the sm_100a tcgen05/TMA kernels of the UNet/TAESD denoiser
against plain PyTorch fp32 references of the same op (bf16 inputs, fp32
accumulation).  Tolerance: relative Frobenius error <= 1e-2 and max-abs
error <= 3e-2 * max|ref| (bf16 output rounding on ~1e2-term dot products)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def K():
    from paper_2312_12491_b200 import _lib

    lib = _lib.lib
    vp, i64 = C.c_void_p, C.c_int64
    lib.sdx_kernel_gemm.argtypes = [vp, i64, vp, i64, vp, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int,
                                    C.c_float, vp]
    lib.sdx_kernel_gemm_concat.argtypes = [vp, i64, C.c_int, vp, i64, vp, i64, vp, C.c_int, C.c_int, C.c_int, vp,
                                           C.c_int, C.c_int, vp]
    lib.sdx_kernel_conv3x3.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp,
                                       C.c_int, vp, C.c_int, vp]
    lib.sdx_kernel_last_error.restype = C.c_char_p
    return lib


def ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def check(got, ref, tol=1e-2):
    got, ref = got.float(), ref.float()
    rel = (got - ref).norm() / ref.norm().clamp_min(1e-6)
    mx = (got - ref).abs().max() / ref.abs().max().clamp_min(1e-6)
    assert rel <= tol and mx <= 3 * tol, (float(rel), float(mx))


def act_ref(x, act):
    return [lambda v: v, torch.nn.functional.silu, torch.relu, torch.nn.functional.gelu][act](x)


@pytest.mark.parametrize("shape", [(256, 320, 320), (300, 640, 1280), (128, 64, 64), (4096, 1280, 2560),
                                   (77, 320, 1024), (1000, 256, 192)])
@pytest.mark.parametrize("act", [0, 1, 3])
@pytest.mark.parametrize("out_f32", [0, 1])
def test_gemm_tc(K, shape, act, out_f32):
    M, N, Kd = shape
    g = torch.Generator(device="cuda").manual_seed(M + N + Kd)
    A = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, Kd, device="cuda", generator=g) / Kd ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.float32 if out_f32 else torch.bfloat16)
    st = K.sdx_kernel_gemm(ptr(A), Kd, ptr(B), Kd, ptr(out), M, N, Kd, ptr(bias), ptr(res), act, out_f32, 1.0,
                           stream())
    assert st == 0, K.sdx_kernel_last_error()
    torch.cuda.synchronize()
    ref = act_ref(A.float() @ B.float().T + bias, act) + res.float()
    check(out, ref)


def test_gemm_concat(K):
    M, N, K1, K2 = 512, 640, 1280, 640
    A1 = torch.randn(M, K1, device="cuda").bfloat16()
    A2 = torch.randn(M, K2, device="cuda").bfloat16()
    B = (torch.randn(N, K1 + K2, device="cuda") / 40).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = K.sdx_kernel_gemm_concat(ptr(A1), K1, K1, ptr(A2), K2, ptr(B), K1 + K2, ptr(out), M, N, K1 + K2, None, 0, 0,
                                  stream())
    assert st == 0, K.sdx_kernel_last_error()
    torch.cuda.synchronize()
    check(out, torch.cat([A1, A2], 1).float() @ B.float().T)


@pytest.mark.parametrize("imgs,H,Cin,Cout,stride", [(2, 64, 64, 320, 1), (1, 64, 320, 320, 1), (3, 32, 128, 640, 1),
                                                    (2, 16, 128, 128, 1), (3, 8, 256, 1280, 1), (2, 64, 64, 64, 2),
                                                    (2, 32, 128, 128, 2), (1, 256, 64, 64, 1), (1, 512, 64, 64, 2)])
def test_conv3x3(K, imgs, H, Cin, Cout, stride):
    W = H
    g = torch.Generator(device="cuda").manual_seed(H * Cin + Cout)
    x = torch.randn(imgs, H, W, Cin, device="cuda", generator=g).bfloat16()
    w = (torch.randn(Cout, 3, 3, Cin, device="cuda", generator=g) / (3 * Cin ** 0.5)).bfloat16()
    bias = torch.randn(Cout, device="cuda", generator=g)
    bimg = torch.randn(imgs, Cout, device="cuda", generator=g)
    Ho = H if stride == 1 else H // 2
    out = torch.empty(imgs, Ho, Ho, Cout, device="cuda", dtype=torch.bfloat16)
    st = K.sdx_kernel_conv3x3(ptr(x), imgs, H, W, Cin, ptr(w), Cout, stride, ptr(bias), ptr(bimg), None, 1, ptr(out),
                              0, stream())
    assert st == 0, K.sdx_kernel_last_error()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.permute(0, 3, 1, 2).float(), w.permute(0, 3, 1, 2).float(), bias, stride, 1)
    ref = ref + bimg[:, :, None, None]
    ref = torch.nn.functional.silu(ref).permute(0, 2, 3, 1)
    check(out, ref)


@pytest.fixture(scope="module")
def KA(K):
    vp, i64 = C.c_void_p, C.c_int64
    K.sdx_kernel_attention.argtypes = [vp, i64, i64, C.c_int, vp, i64, i64, C.c_int, C.c_int, vp, i64, C.c_int,
                                       C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_float, vp]
    return K


@pytest.mark.parametrize("imgs,T,heads", [(2, 4096, 5), (3, 1024, 10), (2, 256, 20), (3, 64, 20), (1, 200, 2)])
def test_self_attention(KA, imgs, T, heads):
    Cd = heads * 64
    g = torch.Generator(device="cuda").manual_seed(T + heads)
    qkv = torch.randn(imgs * T, 3 * Cd, device="cuda", generator=g).bfloat16()
    out = torch.zeros(imgs * T, Cd, device="cuda", dtype=torch.bfloat16)
    st = KA.sdx_kernel_attention(ptr(qkv), imgs * T, 3 * Cd, 0, ptr(qkv), imgs * T, 3 * Cd, Cd, 2 * Cd, ptr(out), Cd,
                                 imgs, heads, T, T, T, None, 0.125, stream())
    assert st == 0, KA.sdx_kernel_last_error()
    torch.cuda.synchronize()
    q, k, v = qkv.float().view(imgs, T, 3, heads, 64).permute(2, 0, 3, 1, 4)
    ref = torch.softmax(q @ k.transpose(-1, -2) * 0.125, -1) @ v  # imgs, heads, T, 64
    check(out, ref.permute(0, 2, 1, 3).reshape(imgs * T, Cd))


@pytest.mark.parametrize("T,heads", [(4096, 5), (256, 20)])
def test_cross_attention(KA, T, heads):
    # 77 prompt tokens padded to 128 keys; images pick prompt 0 or 1 (cond / negative)
    imgs, Cd, P = 3, heads * 64, 2
    g = torch.Generator(device="cuda").manual_seed(7)
    q = torch.randn(imgs * T, Cd, device="cuda", generator=g).bfloat16()
    kv = torch.randn(P * 77, 2 * Cd, device="cuda", generator=g).bfloat16()
    idx = torch.tensor([0, 1, 0], dtype=torch.int32, device="cuda")
    out = torch.zeros(imgs * T, Cd, device="cuda", dtype=torch.bfloat16)
    st = KA.sdx_kernel_attention(ptr(q), imgs * T, Cd, 0, ptr(kv), P * 77, 2 * Cd, 0, Cd, ptr(out), Cd, imgs, heads,
                                 T, 77, 77, ptr(idx), 0.125, stream())
    assert st == 0, KA.sdx_kernel_last_error()
    torch.cuda.synchronize()
    qq = q.float().view(imgs, T, heads, 64).transpose(1, 2)
    kk = kv.float().view(P, 77, 2, heads, 64)
    refs = []
    for i in range(imgs):
        kp, vp_ = kk[idx[i].item(), :, 0].transpose(0, 1), kk[idx[i].item(), :, 1].transpose(0, 1)
        refs.append(torch.softmax(qq[i] @ kp.transpose(-1, -2) * 0.125, -1) @ vp_)
    ref = torch.stack(refs).transpose(1, 2).reshape(imgs * T, Cd)
    check(out, ref)


@pytest.fixture(scope="module")
def KP(K):
    vp, i64 = C.c_void_p, C.c_int64
    K.sdx_kernel_gemm_plan.argtypes = [vp, i64, vp, i64, vp, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.POINTER(vp)]
    K.sdx_kernel_conv3x3_plan.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp, C.c_int,
                                          vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
    K.sdx_kernel_plan_run.argtypes = [vp, C.c_int, vp]
    K.sdx_kernel_plan_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double)]
    K.sdx_kernel_plan_destroy.argtypes = [vp]
    return K


def run_plan(KP, h):
    bn, sp, clk = C.c_int(), C.c_int(), C.c_double()
    assert KP.sdx_kernel_plan_info(h, C.byref(bn), C.byref(sp), C.byref(clk)) == 0
    assert KP.sdx_kernel_plan_run(h, 1, stream()) == 0, KP.sdx_kernel_last_error()
    torch.cuda.synchronize()
    KP.sdx_kernel_plan_destroy(h)
    return bn.value, sp.value


# forced tilings: 1-CTA and CTA-pair (bn < 0, 2-SM tcgen05 MMA), with and without split-K,
# M not a multiple of the 256-row pair tile, residual / bias / ReLU epilogues
@pytest.mark.parametrize("shape", [(16384, 320, 320), (1000, 640, 1280), (300, 256, 2560), (4096, 1280, 640)])
@pytest.mark.parametrize("bn,splits", [(-256, 1), (-160, 1), (-128, 3), (128, 1), (160, 2)])
@pytest.mark.parametrize("act,res", [(0, 1), (2, 0)])
def test_gemm_tilings(KP, shape, bn, splits, act, res):
    M, N, Kd = shape
    g = torch.Generator(device="cuda").manual_seed(M + N + Kd + abs(bn) + splits)
    A = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, Kd, device="cuda", generator=g) / Kd ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    R = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    h = C.c_void_p()
    assert KP.sdx_kernel_gemm_plan(ptr(A), Kd, ptr(B), Kd, ptr(out), M, N, Kd, ptr(bias), ptr(R) if res else None, act,
                                   0, bn, splits, C.byref(h)) == 0, KP.sdx_kernel_last_error()
    got_bn, got_s = run_plan(KP, h)
    assert (got_bn, got_s) == (bn, splits)
    ref = A.float() @ B.float().T + bias
    if act == 2:
        ref = torch.relu(ref)
    if res:
        ref = ref + R.float()
    check(out, ref)


@pytest.mark.parametrize("imgs,H,Cin,Cout,stride,bn,splits", [(4, 64, 320, 320, 1, -160, 1), (3, 32, 640, 640, 1, -256, 1),
                                                           (4, 16, 1280, 1280, 1, -256, 3), (2, 64, 64, 64, 2, -128, 1),
                                                           (1, 512, 64, 64, 1, -128, 1)])
def test_conv3x3_pair(KP, imgs, H, Cin, Cout, stride, bn, splits):
    g = torch.Generator(device="cuda").manual_seed(H * Cin + Cout + 1)
    x = torch.randn(imgs, H, H, Cin, device="cuda", generator=g).bfloat16()
    w = (torch.randn(Cout, 3, 3, Cin, device="cuda", generator=g) / (3 * Cin ** 0.5)).bfloat16()
    bias = torch.randn(Cout, device="cuda", generator=g)
    Ho = H // stride
    out = torch.full((imgs, Ho, Ho, Cout), float("nan"), device="cuda", dtype=torch.bfloat16)
    h = C.c_void_p()
    assert KP.sdx_kernel_conv3x3_plan(ptr(x), imgs, H, H, Cin, ptr(w), Cout, stride, ptr(bias), None, 0, ptr(out), 0, bn,
                                      splits, C.byref(h)) == 0, KP.sdx_kernel_last_error()
    assert run_plan(KP, h) == (bn, splits)
    ref = torch.nn.functional.conv2d(x.permute(0, 3, 1, 2).float(), w.permute(0, 3, 1, 2).float(), bias, stride, 1)
    check(out, ref.permute(0, 2, 3, 1))


# halo-tiled 64 -> 64 conv (TAESD trunk): one 3 x 130-pixel box per 128-pixel tile, nine taps
# as UMMA descriptor offsets, resident weights; bias + residual + ReLU epilogue as TAESD uses it
@pytest.mark.parametrize("imgs,H,W", [(1, 128, 128), (2, 256, 256), (1, 512, 512), (3, 64, 256)])
@pytest.mark.parametrize("act,res", [(2, 1), (0, 0)])
def test_conv3x3_halo(K, imgs, H, W, act, res):
    g = torch.Generator(device="cuda").manual_seed(H * W + imgs + act)
    x = torch.randn(imgs, H, W, 64, device="cuda", generator=g).bfloat16()
    w = (torch.randn(64, 3, 3, 64, device="cuda", generator=g) / 24).bfloat16()
    bias = torch.randn(64, device="cuda", generator=g)
    R = torch.randn(imgs, H, W, 64, device="cuda", generator=g).bfloat16()
    out = torch.full((imgs, H, W, 64), float("nan"), device="cuda", dtype=torch.bfloat16)
    st = K.sdx_kernel_conv3x3(ptr(x), imgs, H, W, 64, ptr(w), 64, 1, ptr(bias), None, ptr(R) if res else None, act,
                              ptr(out), 0, stream())
    assert st == 0, K.sdx_kernel_last_error()
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.permute(0, 3, 1, 2).float(), w.permute(0, 3, 1, 2).float(), bias, 1, 1)
    ref = ref.permute(0, 2, 3, 1)
    if act == 2:
        ref = torch.relu(ref)  # the kernel-level entry applies the activation before the residual
    if res:
        ref = ref + R.float()
    check(out, ref)


@pytest.mark.parametrize("cfg", [(4096, 320, 0, 4, 1), (1024, 640, 640, 2, 1), (64, 1280, 1280, 3, 0),
                                 (256, 1920, 640, 1, 1), (4096, 128, 0, 1, 0)])
@pytest.mark.parametrize("path", ["cluster", "split"])
def test_groupnorm(K, cfg, path, monkeypatch):
    """GroupNorm(32) (+ SiLU) over the channel concat [x1 | x2], NHWC bf16, against
    torch.nn.functional.group_norm in fp32.  Paths: one launch with a 16-CTA cluster
    per image (DSMEM statistics), or statistics (fixed-point atomics) + apply."""
    monkeypatch.setenv("SDX_GN_CLUSTER_MAX", "0" if path == "split" else str(1 << 60))
    HW, C1, C2, imgs, silu = cfg
    vp = C.c_void_p
    K.sdx_kernel_groupnorm.argtypes = [vp, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_float, vp, vp, C.c_int, vp,
                                       vp, C.c_int, vp]
    g = torch.Generator(device="cuda").manual_seed(HW + C1 + C2)
    x1 = (torch.randn(imgs, HW, C1, device="cuda", generator=g) * 2 + 0.5).bfloat16()
    x2 = (torch.randn(imgs, HW, C2, device="cuda", generator=g) - 1).bfloat16() if C2 else None
    Ct = C1 + C2
    gamma = torch.randn(Ct, device="cuda", generator=g)
    beta = torch.randn(Ct, device="cuda", generator=g)
    out = torch.empty(imgs, HW, Ct, device="cuda", dtype=torch.bfloat16)
    arena = torch.zeros(imgs * 64 + 1, device="cuda", dtype=torch.int64)
    st = K.sdx_kernel_groupnorm(ptr(x1), C1, ptr(x2), C2, HW, imgs, 1e-5, ptr(gamma), ptr(beta), silu, ptr(out),
                                ptr(arena), 2, stream())
    assert st == 0, K.sdx_kernel_last_error()
    x = torch.cat([x1, x2], -1) if C2 else x1
    ref = torch.nn.functional.group_norm(x.float().permute(0, 2, 1), 32, gamma, beta, 1e-5).permute(0, 2, 1)
    if silu:
        ref = torch.nn.functional.silu(ref)
    check(out, ref)
