"""Tiling sweep of the tcgen05 GEMM / implicit-GEMM conv on the UNet's layer
shapes: every (BN, split-K) candidate timed with CUDA events over back-to-back
replays of a prebuilt plan, next to the cost model's pick.

    python tools/gemm_sweep.py [rows ...]
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_12491_b200 import _lib  # noqa: E402

L = _lib.lib
vp, i64 = C.c_void_p, C.c_int64
L.sdx_kernel_gemm_plan.argtypes = [vp, i64, vp, i64, vp, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.POINTER(vp)]
L.sdx_kernel_conv3x3_plan.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp, C.c_int, vp,
                                      C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
L.sdx_kernel_plan_run.argtypes = [vp, C.c_int, vp]
L.sdx_kernel_plan_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double)]
L.sdx_kernel_plan_destroy.argtypes = [vp]
L.sdx_kernel_last_error.restype = C.c_char_p
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
BNS = [64, 96, 128, 160, 192, 224, 256, -128, -160, -192, -224, -256]  # < 0: CTA pair
SPLITS = [1, 2, 3, 4, 6, 8, 12, 16]


def time_plan(h, iters=30):
    """Device time per launch: `iters` back-to-back launches captured in one CUDA
    graph (no host launch overhead), replayed 3 times, best replay."""
    assert L.sdx_kernel_plan_run(h, 2, st) == 0, L.sdx_kernel_last_error()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cs = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        assert L.sdx_kernel_plan_run(h, iters, cs) == 0
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / iters)
    return best  # us


def info(h):
    bn, s, clk = C.c_int(), C.c_int(), C.c_double()
    L.sdx_kernel_plan_info(h, C.byref(bn), C.byref(s), C.byref(clk))
    return bn.value, s.value, clk.value


RECORDS = []  # every timed candidate, for fitting the tiling cost model (SDX_SWEEP_JSON)


def sweep(label, make, flops, N, K, M=0, res=False):
    h = vp()
    assert make(0, 0, C.byref(h)) == 0, L.sdx_kernel_last_error()
    mbn, ms, mclk = info(h)
    tm = time_plan(h)
    L.sdx_kernel_plan_destroy(h)
    best = (tm, mbn, ms)
    RECORDS.append({"label": label, "M": M, "N": N, "K": K, "res": res, "bn": mbn, "s": ms, "us": tm, "model": True})
    for bn in ([] if os.environ.get("SDX_SWEEP_MODEL_ONLY") else BNS):
        if N <= 64 and abs(bn) > 64:
            continue
        for s in SPLITS:
            if s > 1 and s > (K // 64) // 4:
                continue
            if (bn, s) == (mbn, ms):
                continue
            h = vp()
            if make(bn, s, C.byref(h)) != 0:
                continue
            t = time_plan(h)
            L.sdx_kernel_plan_destroy(h)
            RECORDS.append({"label": label, "M": M, "N": N, "K": K, "res": res, "bn": bn, "s": s, "us": t,
                            "model": False})
            if t < best[0]:
                best = (t, bn, s)
    print(f"{label:44s} model bn={mbn:3d} s={ms:2d} {tm:7.1f} us ({flops / tm / 1e6:6.1f} TF/s, model {mclk / 1965:6.1f} us)"
          f" | best bn={best[1]:3d} s={best[2]:2d} {best[0]:7.1f} us ({flops / best[0] / 1e6:6.1f} TF/s) x{tm / best[0]:.2f}",
          flush=True)
    return tm, best[0]


def gemm_case(M, N, K, res):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda")
    R = torch.randn(M, N, device="cuda").bfloat16() if res else None
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)

    def make(bn, s, hp):
        return L.sdx_kernel_gemm_plan(A.data_ptr(), K, B.data_ptr(), K, out.data_ptr(), M, N, K, bias.data_ptr(),
                                      R.data_ptr() if res else None, 0, 0, bn, s, hp)

    return sweep(f"linear M={M} N={N} K={K}{' +res' if res else ''}", make, 2.0 * M * N * K, N, K, M, res)


def conv_case(imgs, H, Cin, Cout, stride=1):
    x = torch.randn(imgs, H, H, Cin, device="cuda").bfloat16()
    w = (torch.randn(Cout, 3, 3, Cin, device="cuda") / (3 * Cin ** 0.5)).bfloat16()
    bias = torch.randn(Cout, device="cuda")
    Ho = H // stride
    out = torch.empty(imgs, Ho, Ho, Cout, device="cuda", dtype=torch.bfloat16)

    def make(bn, s, hp):
        return L.sdx_kernel_conv3x3_plan(x.data_ptr(), imgs, H, H, Cin, w.data_ptr(), Cout, stride, bias.data_ptr(),
                                         None, 0, out.data_ptr(), 0, bn, s, hp)

    return sweep(f"conv3x3 {imgs}x{H}^2 {Cin}->{Cout} s{stride}", make, 2.0 * imgs * Ho * Ho * Cout * 9 * Cin, Cout,
                 9 * Cin, imgs * Ho * Ho, False)


def main():
    rows_list = [int(a) for a in sys.argv[1:] if int(a) > 0] if len(sys.argv) > 1 else [4, 8]
    tot_m = tot_b = 0.0
    for R in rows_list:
        print(f"=== rows {R}")
        for hw, C_ in ((4096, 320), (1024, 640), (256, 1280), (64, 1280)):
            M = R * hw
            for (n, k, res) in ((C_, C_, False), (C_, C_, True), (3 * C_, C_, False), (C_, 4 * C_, True)):
                if hw == 64 and C_ == 1280 and R > 0 and False:
                    continue
                a, b = gemm_case(M, n, k, res)
                tot_m += a
                tot_b += b
        for (H, cin, cout) in ((64, 320, 320), (64, 640, 320), (64, 960, 320), (32, 320, 640), (32, 640, 640),
                               (32, 1280, 640), (32, 1920, 640), (16, 640, 1280), (16, 1280, 1280), (16, 2560, 1280),
                               (8, 1280, 1280), (8, 2560, 1280)):
            a, b = conv_case(R, H, cin, cout)
            tot_m += a
            tot_b += b
        for (H, c) in ((64, 320), (32, 640), (16, 1280)):
            a, b = conv_case(R, H, c, c, 2)
            tot_m += a
            tot_b += b
    for (H, cin, cout, s) in ((512, 64, 64, 1), (256, 64, 64, 1), (128, 64, 64, 1), (64, 64, 64, 1), (512, 64, 64, 2),
                              (256, 64, 64, 2), (128, 64, 64, 2)):
        a, b = conv_case(1, H, cin, cout, s)
    print(f"sum over UNet shapes: model {tot_m:.1f} us, best {tot_b:.1f} us")
    if os.environ.get("SDX_SWEEP_JSON"):
        json.dump(RECORDS, open(os.environ["SDX_SWEEP_JSON"], "w"))


if __name__ == "__main__":
    main()
