"""One prebuilt GEMM or conv launched a few times (for ncu captures).

    python tools/one_gemm.py gemm M N K [res] [bn] [splits]
    python tools/one_gemm.py conv imgs H Cin Cout [stride] [bn] [splits]
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
sys.argv += []
from tools.gemm_sweep import L, vp  # noqa: E402

st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
kind, a = sys.argv[1], [int(x) for x in sys.argv[2:]]
h = vp()
if kind == "gemm":
    M, N, K = a[:3]
    res, bn, sp = (a[3:] + [0, 0, 0])[:3]
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    R = torch.randn(M, N, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    assert L.sdx_kernel_gemm_plan(A.data_ptr(), K, B.data_ptr(), K, out.data_ptr(), M, N, K, None,
                                  R.data_ptr() if res else None, 0, 0, bn, sp, C.byref(h)) == 0
else:
    imgs, H, cin, cout = a[:4]
    stride, bn, sp = (a[4:] + [1, 0, 0])[:3] if len(a) > 4 else (1, 0, 0)
    x = torch.randn(imgs, H, H, cin, device="cuda").bfloat16()
    w = (torch.randn(cout, 3, 3, cin, device="cuda") / (3 * cin ** 0.5)).bfloat16()
    out = torch.empty(imgs, H // stride, H // stride, cout, device="cuda", dtype=torch.bfloat16)
    assert L.sdx_kernel_conv3x3_plan(x.data_ptr(), imgs, H, H, cin, w.data_ptr(), cout, stride, None, None, 0,
                                     out.data_ptr(), 0, bn, sp, C.byref(h)) == 0
assert L.sdx_kernel_plan_run(h, 5, st) == 0
torch.cuda.synchronize()
print("ok")
