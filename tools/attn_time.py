"""Graph-timed attention launches at the UNet's shapes (self-attention T=4096/1024/256,
cross-attention), for A/B runs of the kernel variants (SDX_ATTN_TS=0|1).

    python tools/attn_time.py
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_12491_b200 import _lib  # noqa: E402

L = _lib.lib
vp, i64 = C.c_void_p, C.c_int64
L.sdx_kernel_attention.argtypes = [vp, i64, i64, C.c_int, vp, i64, i64, C.c_int, C.c_int, vp, i64, C.c_int, C.c_int,
                                   C.c_int, C.c_int, C.c_int, vp, C.c_float, vp]


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


tag = "ts" if os.environ.get("SDX_ATTN_TS", "1") != "0" else "smemP"
for imgs, T, heads, kv in ((4, 4096, 5, 0), (8, 4096, 5, 0), (4, 1024, 10, 0), (8, 1024, 10, 0), (4, 256, 20, 0),
                           (4, 4096, 5, 77)):
    Cd = heads * 64
    qkv = torch.randn(imgs * T, 3 * Cd, device="cuda").bfloat16()
    out = torch.zeros(imgs * T, Cd, device="cuda", dtype=torch.bfloat16)
    if kv:
        kvb = torch.randn(128, 2 * Cd, device="cuda").bfloat16()
        idx = torch.zeros(imgs, dtype=torch.int32, device="cuda")
        fn = lambda s: L.sdx_kernel_attention(qkv.data_ptr(), imgs * T, 3 * Cd, 0, kvb.data_ptr(), 128, 2 * Cd, 0,  # noqa
                                              Cd, out.data_ptr(), Cd, imgs, heads, T, kv, 128, idx.data_ptr(), 0.125, s)
        fl = 4.0 * imgs * heads * T * kv * 64
    else:
        fn = lambda s: L.sdx_kernel_attention(qkv.data_ptr(), imgs * T, 3 * Cd, 0, qkv.data_ptr(), imgs * T, 3 * Cd,  # noqa
                                              Cd, 2 * Cd, out.data_ptr(), Cd, imgs, heads, T, T, T, None, 0.125, s)
        fl = 4.0 * imgs * heads * T * T * 64
    us = timed(fn)
    print(f"[{tag}] attn imgs={imgs} T={T} heads={heads} kv={kv or T}: {us:8.1f} us  {fl / us / 1e6:7.1f} TF/s", flush=True)
