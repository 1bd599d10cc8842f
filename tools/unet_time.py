"""Device time of whole UNet forwards (one CUDA graph replayed back to back; the
weights stream from HBM every forward as in the pipeline), at the given row counts.

    python tools/unet_time.py [rows ...]
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2312_12491_b200 import _lib  # noqa: E402

L = _lib.lib
vp = C.c_void_p
L.sdx_kernel_last_error.restype = C.c_char_p
L.sdx_unet_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.c_uint64, C.c_int, C.POINTER(vp)]
L.sdx_unet_time_forward.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_float)]
L.sdx_unet_flops_per_row.argtypes = [vp, C.POINTER(C.c_double)]
rows_list = [int(a) for a in sys.argv[1:]] or [4, 8]
taus = (C.c_int * 4)(999, 749, 499, 249)
h = vp()
assert L.sdx_unet_create(max(rows_list), taus, 4, 1234, 0, C.byref(h)) == 0, L.sdx_kernel_last_error()
f = C.c_double()
L.sdx_unet_flops_per_row(h, C.byref(f))
for r in rows_list:
    ms = C.c_float()
    best = 1e9
    for _ in range(3):
        assert L.sdx_unet_time_forward(h, r, 20, C.byref(ms)) == 0, L.sdx_kernel_last_error()
        best = min(best, ms.value)
    print(f"UNet forward rows={r}: {best:.3f} ms ({r * f.value / best / 1e9:.1f} TFLOP/s)")
