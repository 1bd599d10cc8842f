"""The device TAESD-class codec (halo-tiled tcgen05 64->64 convs, direct CUDA-core
RGB input conv, bf16 activations, fp32 accumulation) against its PyTorch fp32
restatement with the same weights (read back through sdx_taesd_param):

  encoder  u8/255 -> conv 3->64 -> block -> [down (stride 2, no bias) -> 3 blocks] x 3 -> conv 64->4
  decoder  tanh(z/3)*3 -> conv 4->64 + ReLU -> 3 blocks -> [nearest 2x -> conv (no bias) -> blocks] x 3
           -> conv 64->3 -> round(255 clamp(., 0, 1))
  block    relu(c2(relu(c1(relu(c0(x))))) + x)

Tolerances (bf16 activations through ~30 convs): encoder latents relative Frobenius
<= 3e-2; decoder frames mean |diff| <= 1.5 levels and >= 97% within 4 levels of 255."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
F = pytest.importorskip("torch.nn.functional")


@pytest.fixture(scope="module")
def taesd():
    from paper_2312_12491_b200 import _lib

    L = _lib.lib
    vp = C.c_void_p
    L.sdx_taesd_create.argtypes = [C.c_int, C.c_uint64, C.c_int, C.POINTER(vp)]
    L.sdx_taesd_destroy.argtypes = [vp]
    L.sdx_taesd_encode.argtypes = [vp, vp, C.c_int, vp, vp]
    L.sdx_taesd_decode.argtypes = [vp, vp, C.c_int, vp, vp]
    L.sdx_taesd_param_count.argtypes = [vp, C.POINTER(C.c_int)]
    L.sdx_taesd_param.argtypes = [vp, C.c_int, C.POINTER(C.c_char_p), C.POINTER(vp), C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.sdx_memcpy_d2d.argtypes = [vp, vp, C.c_int64]
    L.sdx_kernel_last_error.restype = C.c_char_p
    h = vp()
    assert L.sdx_taesd_create(3, 77, 0, C.byref(h)) == 0, L.sdx_kernel_last_error()
    n = C.c_int()
    assert L.sdx_taesd_param_count(h, C.byref(n)) == 0
    params = {}
    for i in range(n.value):
        name, ptr, shape, nd, f32 = C.c_char_p(), vp(), (C.c_int64 * 4)(), C.c_int(), C.c_int()
        assert L.sdx_taesd_param(h, i, C.byref(name), C.byref(ptr), shape, C.byref(nd), C.byref(f32)) == 0
        shp = [shape[k] for k in range(nd.value)]
        t = torch.empty(shp, device="cuda", dtype=torch.float32 if f32.value else torch.bfloat16)
        L.sdx_memcpy_d2d(C.c_void_p(t.data_ptr()), ptr, t.numel() * t.element_size())
        params[name.value.decode()] = t.float()
    torch.cuda.synchronize()
    yield L, h, params
    L.sdx_taesd_destroy(h)


def conv(x, w, b=None, stride=1):
    # x NCHW fp32, w [Cout][3][3][Cin] (device layout)
    return F.conv2d(x, w.permute(0, 3, 1, 2), b, stride, 1)


def block(P, x, nm):
    a = F.relu(conv(x, P[nm + ".c0.w"], P[nm + ".c0.b"]))
    b = F.relu(conv(a, P[nm + ".c1.w"], P[nm + ".c1.b"]))
    return F.relu(conv(b, P[nm + ".c2.w"], P[nm + ".c2.b"]) + x)


def encode_ref(P, frames):
    x = frames.float().permute(0, 3, 1, 2) / 255.0
    w_in = P["enc.conv_in.w"][:, :27].reshape(64, 3, 3, 3)  # column k = tap * 3 + c
    x = conv(x, w_in, P["enc.conv_in.b"])
    x = block(P, x, "enc.b0")
    for r in range(1, 4):
        x = conv(x, P[f"enc.down{r}.w"], None, 2)
        for j in range(3):
            x = block(P, x, f"enc.b{r}{j}")
    return conv(x, P["enc.conv_out.w"], P["enc.conv_out.b"]).permute(0, 2, 3, 1)


def decode_ref(P, lat):
    x = torch.tanh(lat.permute(0, 3, 1, 2) / 3.0) * 3.0
    w_in = P["dec.conv_in.w"][:, :36].reshape(64, 3, 3, 4)
    x = F.relu(conv(x, w_in, P["dec.conv_in.b"]))
    for j in range(3):
        x = block(P, x, f"dec.b3{j}")
    for r in (2, 1, 0):
        x = F.interpolate(x, scale_factor=2, mode="nearest")
        x = conv(x, P[f"dec.up{r}.w"])
        for j in range(1 if r == 0 else 3):
            x = block(P, x, f"dec.b{r}{j}")
    y = conv(x, P["dec.conv_out.w"], P["dec.conv_out.b"]).permute(0, 2, 3, 1)
    return torch.round(y.clamp(0, 1) * 255.0)


def frames_u8(n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    yy, xx = torch.meshgrid(torch.arange(512, device="cuda"), torch.arange(512, device="cuda"), indexing="ij")
    out = []
    for i in range(n):
        base = torch.stack([(xx + 40 * i) % 256, (yy * 2 + 17 * i) % 256, (xx + yy) % 256], -1).float()
        noise = torch.randint(0, 40, (512, 512, 3), device="cuda", generator=g).float()
        out.append((base * 0.8 + noise).clamp(0, 255))
    return torch.stack(out).to(torch.uint8).contiguous()


@pytest.mark.parametrize("n", [1, 3])
def test_taesd_encoder_matches_torch_fp32(taesd, n):
    L, h, P = taesd
    fr = frames_u8(n, 5 + n)
    lat = torch.empty(n, 64, 64, 4, device="cuda")
    assert L.sdx_taesd_encode(h, C.c_void_p(fr.data_ptr()), n, C.c_void_p(lat.data_ptr()), None) == 0, \
        L.sdx_kernel_last_error()
    ref = encode_ref(P, fr)
    rel = float((lat - ref).norm() / ref.norm())
    assert rel <= 3e-2, rel
    for i in range(n):  # per image: each image goes to its own latent block
        assert float(torch.nn.functional.cosine_similarity(lat[i].flatten(), ref[i].flatten(), dim=0)) >= 0.999


@pytest.mark.parametrize("n", [1, 2])
def test_taesd_decoder_matches_torch_fp32(taesd, n):
    L, h, P = taesd
    g = torch.Generator(device="cuda").manual_seed(11 + n)
    lat = torch.randn(n, 64, 64, 4, device="cuda", generator=g)
    fr = torch.empty(n, 512, 512, 3, device="cuda", dtype=torch.uint8)
    assert L.sdx_taesd_decode(h, C.c_void_p(lat.data_ptr()), n, C.c_void_p(fr.data_ptr()), None) == 0, \
        L.sdx_kernel_last_error()
    ref = decode_ref(P, lat)
    diff = (fr.float() - ref).abs()
    assert float(diff.mean()) <= 1.5, float(diff.mean())
    assert float((diff <= 4).float().mean()) >= 0.97
    assert float(ref.std()) > 10.0  # the random decoder produces a non-trivial image
