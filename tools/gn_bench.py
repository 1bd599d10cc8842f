"""GroupNorm kernel timing on the UNet's shapes at R rows: `iters` passes
(arena zero + statistics + apply) captured in one CUDA graph, best of 3
replays, next to the bytes each pass moves (read twice, write once).

    python tools/gn_bench.py [rows]
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_12491_b200 import _lib  # noqa: E402

L = _lib.lib
vp = C.c_void_p
L.sdx_kernel_groupnorm.argtypes = [vp, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_float, vp, vp, C.c_int, vp, vp,
                                   C.c_int, vp]
L.sdx_kernel_last_error.restype = C.c_char_p


def run(HW, C1, C2, imgs, iters):
    x1 = torch.randn(imgs, HW, C1, device="cuda").bfloat16()
    x2 = torch.randn(imgs, HW, C2, device="cuda").bfloat16() if C2 else None
    gm = torch.ones(C1 + C2, device="cuda")
    bt = torch.zeros(C1 + C2, device="cuda")
    out = torch.empty(imgs, HW, C1 + C2, device="cuda", dtype=torch.bfloat16)
    ar = torch.zeros(imgs * 64 + 1, device="cuda", dtype=torch.int64)
    p = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731

    def go(n):
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        assert L.sdx_kernel_groupnorm(p(x1), C1, p(x2), C2, HW, imgs, 1e-5, p(gm), p(bt), 1, p(out), p(ar), n, s) == 0, \
            L.sdx_kernel_last_error()

    go(2)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        go(iters)
    best = 1e30
    for _ in range(3):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / iters)
    return best


def main():
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    shapes = [(4096, 320, 0), (4096, 320, 320), (4096, 320, 640), (1024, 640, 0), (1024, 640, 320), (1024, 640, 640),
              (1024, 1280, 0), (256, 1280, 0), (256, 1280, 640), (256, 1280, 1280), (256, 2560, 0), (64, 1280, 0),
              (64, 1280, 1280)]
    for HW, C1, C2 in shapes:
        os.environ["SDX_GN_PARTS"] = "6"
        os.environ["SDX_GN_CLUSTER_MAX"] = str(1 << 60)
        cl = run(HW, C1, C2, R, 20)
        os.environ["SDX_GN_CLUSTER_SIZE"] = "8"
        cl8 = run(HW, C1, C2, R, 20)
        os.environ["SDX_GN_CLUSTER_SIZE"] = "16"
        cl4 = run(HW, C1, C2, R, 20)
        os.environ.pop("SDX_GN_CLUSTER_SIZE")
        os.environ["SDX_GN_CLUSTER_MAX"] = "0"
        parts = {}
        for k, v in (("zero", "1"), ("stats", "2"), ("apply", "4"), ("all", "7")):
            os.environ["SDX_GN_PARTS"] = v
            parts[k] = run(HW, C1, C2, R, 20)
        us = parts["all"]
        mb = R * HW * (C1 + C2) * 2 * 3 / 1e6
        print(f"GN HW={HW:5d} C={C1}+{C2:4d} imgs={R}: {us:6.2f} us  ({mb:6.2f} MB, {mb / us:6.2f} TB/s)  "
              f"zero {parts['zero']:5.2f} stats {parts['stats']:5.2f} apply {parts['apply']:5.2f} | cluster default {cl:6.2f} 8 {cl8:6.2f} 16 {cl4:6.2f} us", flush=True)


if __name__ == "__main__":
    main()
