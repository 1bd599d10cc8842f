"""Attention pipeline probes: full vs no-MMA vs no-softmax-math, graph-timed.

    python tools/attn_probe.py
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_12491_b200 import _lib  # noqa: E402

L = _lib.lib
vp, i64 = C.c_void_p, C.c_int64
L.sdx_kernel_attention.argtypes = [vp, i64, i64, C.c_int, vp, i64, i64, C.c_int, C.c_int, vp, i64, C.c_int, C.c_int,
                                   C.c_int, C.c_int, C.c_int, vp, C.c_float, vp]
L.sdx_kernel_attention_probe.argtypes = [C.c_int]


def timed(fn, iters=20):
    fn(C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cs = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for _ in range(iters):
            fn(cs)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / iters


for imgs, T, heads in ((4, 4096, 5), (8, 4096, 5), (4, 1024, 10)):
    Cd = heads * 64
    qkv = torch.randn(imgs * T, 3 * Cd, device="cuda").bfloat16()
    out = torch.zeros(imgs * T, Cd, device="cuda", dtype=torch.bfloat16)
    fn = lambda s: L.sdx_kernel_attention(qkv.data_ptr(), imgs * T, 3 * Cd, 0, qkv.data_ptr(), imgs * T, 3 * Cd, Cd,  # noqa
                                          2 * Cd, out.data_ptr(), Cd, imgs, heads, T, T, T, None, 0.125, s)
    res = []
    for mode in (0, 1, 2, 5, 6, 7):
        L.sdx_kernel_attention_probe(mode)
        res.append(timed(fn))
    L.sdx_kernel_attention_probe(0)
    fl = 4.0 * imgs * heads * T * T * 64
    print(f"attn imgs={imgs} T={T} heads={heads}: full {res[0]:7.1f} us ({fl / res[0] / 1e6:6.1f} TF/s) | no-mma {res[1]:7.1f} | no-softmax {res[2]:7.1f} | no-PV {res[3]:7.1f} | no-S {res[4]:7.1f} | skeleton {res[5]:7.1f}", flush=True)
