"""Per-CTA phase timeline of one GEMM / conv launch (%globaltimer stamps):
entry, setup done, first K-slice landed, first tile committed, epilogue of the
first tile start / end, exit.  Prints min / median / max over CTAs in us,
relative to the earliest CTA entry, plus the event-timed launch duration.

    python tools/gemm_phases.py
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from tools.gemm_sweep import L, vp  # noqa: E402

L.sdx_kernel_gemm_debug.argtypes = [vp]
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
NAMES = ["entry", "setup", "1st stage", "1st commit", "epi start", "epi end", "exit", "c0 tmem", "c0 slab", "c0 pass",
         "c1 tmem", "c1 slab", "c1 pass"]


def run(label, make):
    h = vp()
    assert make(C.byref(h)) == 0, L.sdx_kernel_last_error()
    dbg = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
    for _ in range(3):
        L.sdx_kernel_plan_run(h, 1, st)
    torch.cuda.synchronize()
    L.sdx_kernel_gemm_debug(C.c_void_p(dbg.data_ptr()))
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    L.sdx_kernel_plan_run(h, 1, st)
    b.record()
    torch.cuda.synchronize()
    L.sdx_kernel_gemm_debug(None)
    d = dbg.view(148, 16)[:, :13].cpu()
    live = d[:, 0] > 0
    d = d[live].double()
    t0 = d[:, 0].min()
    rel = (d - t0) / 1000.0
    print(f"{label}: {int(live.sum())} CTAs, event {a.elapsed_time(b) * 1e3:.1f} us, span {(d[:, 6].max() - t0) / 1e3:.1f} us")
    for i, n in enumerate(NAMES):
        col = rel[:, i]
        col = col[d[:, i] > 0]
        if len(col):
            print(f"   {n:10s} min {col.min():7.2f} med {col.median():7.2f} max {col.max():7.2f}")
    L.sdx_kernel_plan_destroy(h)


def gemm(M, N, K, res=False, bn=0, s=0):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    R = torch.randn(M, N, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    run(f"gemm {M}x{N}x{K}{' +res' if res else ''} bn={bn} s={s}",
        lambda hp: L.sdx_kernel_gemm_plan(A.data_ptr(), K, B.data_ptr(), K, out.data_ptr(), M, N, K, None,
                                          R.data_ptr() if res else None, 0, 0, bn, s, hp))


def conv(imgs, H, cin, cout, stride=1):
    x = torch.randn(imgs, H, H, cin, device="cuda").bfloat16()
    w = (torch.randn(cout, 3, 3, cin, device="cuda") / (3 * cin ** 0.5)).bfloat16()
    out = torch.empty(imgs, H // stride, H // stride, cout, device="cuda", dtype=torch.bfloat16)
    run(f"conv {imgs}x{H}^2 {cin}->{cout} s{stride}",
        lambda hp: L.sdx_kernel_conv3x3_plan(x.data_ptr(), imgs, H, H, cin, w.data_ptr(), cout, stride, None, None, 0,
                                             out.data_ptr(), 0, 0, 0, hp))


if len(sys.argv) > 1 and sys.argv[1] == "taesd":
    conv(8, 512, 64, 64)
    conv(1, 512, 64, 64)
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "small":
    # the UNet's small-K linears at 4 rows
    gemm(16384, 320, 320, True)
    gemm(1024, 1280, 1280, True)
    gemm(4096, 640, 640, True)
    gemm(1024, 1280, 1280)
else:
    conv(4, 64, 320, 320)
    conv(4, 32, 640, 640)
    gemm(16384, 320, 1280, True)
    gemm(8192, 8192, 8192)
