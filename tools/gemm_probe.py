"""Pipeline probes of the tcgen05 GEMM: full kernel vs TMA-only (no MMAs) vs
MMA-only (no loads), graph-timed, for a few UNet shapes and tilings.

    python tools/gemm_probe.py
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from tools.gemm_sweep import L, time_plan, vp  # noqa: E402

L.sdx_kernel_gemm_probe.argtypes = [C.c_int]


def probe(label, make, flops):
    res = []
    for mode in (0, 1, 2, 4):
        L.sdx_kernel_gemm_probe(mode)
        h = vp()
        assert make(C.byref(h)) == 0, L.sdx_kernel_last_error()
        res.append(time_plan(h))
        L.sdx_kernel_plan_destroy(h)
    L.sdx_kernel_gemm_probe(0)
    print(f"{label:48s} full {res[0]:7.1f} us ({flops / res[0] / 1e6:6.1f} TF/s) | tma-only {res[1]:7.1f} | mma-only {res[2]:7.1f}"
          f" | no-epilogue {res[3]:7.1f}",
          flush=True)


def conv(imgs, H, cin, cout, bn, s=1):
    x = torch.randn(imgs, H, H, cin, device="cuda").bfloat16()
    w = (torch.randn(cout, 3, 3, cin, device="cuda") / (3 * cin ** 0.5)).bfloat16()
    out = torch.empty(imgs, H, H, cout, device="cuda", dtype=torch.bfloat16)
    probe(f"conv {imgs}x{H}^2 {cin}->{cout} bn={bn} s={s}",
          lambda hp: L.sdx_kernel_conv3x3_plan(x.data_ptr(), imgs, H, H, cin, w.data_ptr(), cout, 1, None, None, 0,
                                               out.data_ptr(), 0, bn, s, hp), 2.0 * imgs * H * H * cout * 9 * cin)


def gemm(M, N, K, bn, s=1):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    probe(f"gemm {M}x{N}x{K} bn={bn} s={s}",
          lambda hp: L.sdx_kernel_gemm_plan(A.data_ptr(), K, B.data_ptr(), K, out.data_ptr(), M, N, K, None, None, 0,
                                            0, bn, s, hp), 2.0 * M * N * K)


if len(sys.argv) > 1 and sys.argv[1] == "taesd":  # halo-tiled 64 -> 64 convs
    for imgs, H in ((1, 512), (8, 512), (1, 256), (8, 256), (1, 128)):
        conv(imgs, H, 64, 64, 0)
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "bn":
    for bn in (64, 96, 128, 160, 192, 224, 256, -128, -160, -256):
        gemm(8192, 8192, 4096, bn)
    for bn in (64, 128, 160, 192, 256, -256):
        conv(8, 64, 640, 640, bn)
    sys.exit(0)
for bn in (160, 192, 256, -160, -256):
    conv(4, 64, 320, 320, bn)
for bn in (160, 256, -256):
    conv(4, 32, 1280, 640, bn)
for bn in (256, -256):
    gemm(8192, 8192, 8192, bn)
    gemm(16384, 1280, 1280, bn)
for bn in (160, -160):
    gemm(16384, 320, 1280, bn)
