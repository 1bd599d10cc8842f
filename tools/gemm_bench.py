"""Times the tcgen05 GEMM / conv kernels on UNet shapes vs cuBLAS (torch.matmul), CUDA events."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_12491_b200 import _lib  # noqa: E402

L = _lib.lib
vp, i64 = C.c_void_p, C.c_int64
L.sdx_kernel_gemm.argtypes = [vp, i64, vp, i64, vp, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int, C.c_float, vp]
L.sdx_kernel_conv3x3.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp, C.c_int, vp,
                                 C.c_int, vp]


def t(fn, it=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for (M, N, K) in [(8192, 8192, 8192), (16384, 960, 320), (16384, 2560, 320), (16384, 320, 1280), (16384, 320, 320),
                  (4096, 1920, 640), (4096, 640, 2560), (1024, 3840, 1280), (1024, 1280, 5120)]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ms = t(lambda: L.sdx_kernel_gemm(A.data_ptr(), K, B.data_ptr(), K, out.data_ptr(), M, N, K, None, None, 0, 0, 1.0, st))
    ms_cb = t(lambda: torch.matmul(A, B.T))
    f = 2 * M * N * K
    print(f"gemm {M}x{N}x{K}: ours {ms*1e3:8.1f} us {f/ms/1e9:7.1f} TF/s | cublas {ms_cb*1e3:8.1f} us {f/ms_cb/1e9:7.1f} TF/s")
for (imgs, Hh, Cin, Cout) in [(4, 64, 320, 320), (4, 32, 640, 640), (4, 16, 1280, 1280), (4, 8, 1280, 1280),
                              (1, 512, 64, 64), (1, 256, 64, 64)]:
    x = torch.randn(imgs, Hh, Hh, Cin, device="cuda").bfloat16()
    w = torch.randn(Cout, 3, 3, Cin, device="cuda").bfloat16()
    out = torch.empty(imgs, Hh, Hh, Cout, device="cuda", dtype=torch.bfloat16)
    ms = t(lambda: L.sdx_kernel_conv3x3(x.data_ptr(), imgs, Hh, Hh, Cin, w.data_ptr(), Cout, 1, None, None, None, 0,
                                        out.data_ptr(), 0, st))
    xc = x.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
    wc = w.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
    ms_cd = t(lambda: torch.nn.functional.conv2d(xc, wc, None, 1, 1))
    f = 2 * imgs * Hh * Hh * Cout * 9 * Cin
    print(f"conv {imgs}x{Hh}^2 {Cin}->{Cout}: ours {ms*1e3:8.1f} us {f/ms/1e9:7.1f} TF/s | cudnn {ms_cd*1e3:8.1f} us {f/ms_cd/1e9:7.1f} TF/s")
