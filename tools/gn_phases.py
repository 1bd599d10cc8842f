"""Per-CTA phase timeline of the cluster GroupNorm kernel (%globaltimer stamps):
entry, after the PDL wait, first piece landed, statistics summed, cluster barrier,
group statistics, apply done, exit.  The last of `chain` back-to-back launches in one
CUDA graph is stamped (so the kernel runs behind its own predecessor, as in the forward).

    python tools/gn_phases.py [HW C imgs]
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
L.sdx_kernel_groupnorm_debug.argtypes = [vp]
L.sdx_kernel_last_error.restype = C.c_char_p
NAMES = ["entry", "pdl wait", "1st piece", "stats", "cl barrier", "group stats", "apply", "exit"]


def main():
    HW, C1, imgs = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 320, 4)
    os.environ["SDX_GN_PARTS"] = "6"
    x1 = torch.randn(imgs, HW, C1, device="cuda").bfloat16()
    gm, bt = torch.ones(C1, device="cuda"), torch.zeros(C1, device="cuda")
    out = torch.empty(imgs, HW, C1, device="cuda", dtype=torch.bfloat16)
    ar = torch.zeros(imgs * 64 + 1, device="cuda", dtype=torch.int64)
    dbg = torch.zeros(imgs * 16 * 8, device="cuda", dtype=torch.int64)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    go = lambda n: L.sdx_kernel_groupnorm(p(x1), C1, None, 0, HW, imgs, 1e-5, p(gm), p(bt), 1, p(out), p(ar), n, s)  # noqa
    assert go(3) == 0, L.sdx_kernel_last_error()
    torch.cuda.synchronize()
    for chain in (1, 8):
        L.sdx_kernel_groupnorm_debug(p(dbg))
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        assert go(chain) == 0
        b.record()
        torch.cuda.synchronize()
        L.sdx_kernel_groupnorm_debug(None)
        d = dbg.view(-1, 8).cpu().double()
        d = d[d[:, 0] > 0]
        t0 = d[:, 0].min()
        rel = (d - t0) / 1000.0
        print(f"GN HW={HW} C={C1} imgs={imgs}, chain of {chain}: {len(d)} CTAs, {a.elapsed_time(b) * 1e3 / chain:.1f} us"
              f" per launch (event), last launch span {(d[:, 7].max() - t0) / 1e3:.2f} us")
        for i, n in enumerate(NAMES):
            col = rel[:, i]
            print(f"   {n:12s} min {col.min():6.2f} med {col.median():6.2f} max {col.max():6.2f}")


if __name__ == "__main__":
    main()
