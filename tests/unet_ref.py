"""TEST INFRASTRUCTURE: plain PyTorch fp32 restatement of the device UNet
(paper_2312_12491_b200/csrc/unet.cu) evaluated with the device's own
(bf16-rounded) weights, exported through sdx_unet_param.  The UNet has no
reference implementation in /root/reference (parity unpinned at
the UNet level); this fp32 restatement of the declared topology is its oracle.
"""
import ctypes as C
import math

import torch
import torch.nn.functional as F


def export_params(lib, h):
    n = C.c_int()
    assert lib.sdx_unet_param_count(h, C.byref(n)) == 0
    out = {}
    for i in range(n.value):
        name, ptr = C.c_char_p(), C.c_void_p()
        shape = (C.c_int64 * 4)()
        nd, f32 = C.c_int(), C.c_int()
        assert lib.sdx_unet_param(h, i, C.byref(name), C.byref(ptr), shape, C.byref(nd), C.byref(f32)) == 0
        shp = [shape[k] for k in range(nd.value)]
        t = torch.empty(shp, device="cuda", dtype=torch.float32 if f32.value else torch.bfloat16)
        assert lib.sdx_memcpy_d2d(C.c_void_p(t.data_ptr()), ptr, t.numel() * t.element_size()) == 0
        out[name.value.decode()] = t.float()
    return out


def timestep_embedding(taus, dim=320):
    half = dim // 2
    f = torch.exp(-math.log(10000.0) * torch.arange(half, device=taus.device, dtype=torch.float32) / half)
    a = taus.float()[:, None] * f[None]
    return torch.cat([torch.cos(a), torch.sin(a)], -1)


def conv(x, w, b, stride=1):  # x NCHW, w [Cout,3,3,Cin]
    return F.conv2d(x, w.permute(0, 3, 1, 2), b, stride, 1)


def gn(x, g, b, eps, silu):
    y = F.group_norm(x, 32, g, b, eps)
    return F.silu(y) if silu else y


def unet_forward(P, x, taus, prompts, levels=(320, 640, 1280, 1280)):
    """x: [R,64,64,4] fp32 NHWC; taus: [R] timesteps; prompts: [R] prompt index."""
    R = x.shape[0]
    e1 = F.silu(timestep_embedding(taus) @ P["time.linear1.w"].T + P["time.linear1.b"])
    temb = F.silu(e1 @ P["time.linear2.w"].T + P["time.linear2.b"])
    ctx = P["context"]

    def resblock(h, skip, nm):
        inp = torch.cat([h, skip], 1) if skip is not None else h
        t = gn(inp, P[nm + ".norm1.g"], P[nm + ".norm1.b"], 1e-5, True)
        y = conv(t, P[nm + ".conv1.w"], P[nm + ".conv1.b"])
        y = y + (temb @ P[nm + ".temb.w"].T + P[nm + ".temb.b"])[:, :, None, None]
        t2 = gn(y, P[nm + ".norm2.g"], P[nm + ".norm2.b"], 1e-5, True)
        if nm + ".short.w" in P:
            sc = F.conv2d(inp, P[nm + ".short.w"][:, :, None, None], P[nm + ".short.b"])
        else:
            sc = h
        return conv(t2, P[nm + ".conv2.w"], P[nm + ".conv2.b"]) + sc

    def attn(q, k, v, heads):
        B, T, Cc = q.shape
        q = q.view(B, T, heads, 64).transpose(1, 2)
        k = k.reshape(B, -1, heads, 64).transpose(1, 2)
        v = v.reshape(B, -1, heads, 64).transpose(1, 2)
        o = torch.softmax(q @ k.transpose(-1, -2) * 0.125, -1) @ v
        return o.transpose(1, 2).reshape(B, T, Cc)

    def transformer(h, nm):
        B, Cc, H, W = h.shape
        heads = Cc // 64
        t = gn(h, P[nm + ".norm.g"], P[nm + ".norm.b"], 1e-6, False)
        t = t.permute(0, 2, 3, 1).reshape(B, H * W, Cc)
        x1 = t @ P[nm + ".proj_in.w"].T + P[nm + ".proj_in.b"]
        n1 = F.layer_norm(x1, (Cc,), P[nm + ".ln1.g"], P[nm + ".ln1.b"], 1e-5)
        qkv = n1 @ P[nm + ".attn1.qkv.w"].T
        a = attn(qkv[..., :Cc], qkv[..., Cc:2 * Cc], qkv[..., 2 * Cc:], heads)
        x2 = a @ P[nm + ".attn1.out.w"].T + P[nm + ".attn1.out.b"] + x1
        n2 = F.layer_norm(x2, (Cc,), P[nm + ".ln2.g"], P[nm + ".ln2.b"], 1e-5)
        q = n2 @ P[nm + ".attn2.q.w"].T
        kv = ctx[prompts] @ P[nm + ".attn2.kv.w"].T  # [B,77,2C]
        a2 = attn(q, kv[..., :Cc], kv[..., Cc:], heads)
        x3 = a2 @ P[nm + ".attn2.out.w"].T + P[nm + ".attn2.out.b"] + x2
        n3 = F.layer_norm(x3, (Cc,), P[nm + ".ln3.g"], P[nm + ".ln3.b"], 1e-5)
        ff = n3 @ P[nm + ".ff1.w"].T + P[nm + ".ff1.b"]
        u = ff[..., :4 * Cc] * F.gelu(ff[..., 4 * Cc:])
        x4 = u @ P[nm + ".ff2.w"].T + P[nm + ".ff2.b"] + x3
        out = x4 @ P[nm + ".proj_out.w"].T + P[nm + ".proj_out.b"]
        return out.reshape(B, H, W, Cc).permute(0, 3, 1, 2) + h

    xc = x.permute(0, 3, 1, 2)
    w_in = P["conv_in.w"][:, :36].reshape(-1, 3, 3, 4)
    h = conv(xc, w_in, P["conv_in.b"])
    skips = [h]
    attn_lv = [True, True, True, False]
    for l in range(4):
        for j in range(2):
            h = resblock(h, None, f"down{l}.res{j}")
            if attn_lv[l]:
                h = transformer(h, f"down{l}.attn{j}")
            skips.append(h)
        if l < 3:
            h = conv(h, P[f"down{l}.down.w"], P[f"down{l}.down.b"], 2)
            skips.append(h)
    h = resblock(h, None, "mid.res0")
    h = transformer(h, "mid.attn0")
    h = resblock(h, None, "mid.res1")
    for u in range(4):
        l = 3 - u
        for j in range(3):
            h = resblock(h, skips.pop(), f"up{u}.res{j}")
            if attn_lv[l]:
                h = transformer(h, f"up{u}.attn{j}")
        if l > 0:
            h = F.interpolate(h, scale_factor=2, mode="nearest")
            h = conv(h, P[f"up{u}.up.w"], P[f"up{u}.up.b"])
    t = gn(h, P["norm_out.g"], P["norm_out.b"], 1e-5, True)
    eps = conv(t, P["conv_out.w"], P["conv_out.b"])
    return eps.permute(0, 2, 3, 1)
