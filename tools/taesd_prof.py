"""Per-op device times of the TAESD encoder and decoder (each op alone, graph-timed),
at the given image counts.

    python tools/taesd_prof.py [images ...]
"""
import collections
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2312_12491_b200 import _lib  # noqa: E402

L = _lib.lib
vp = C.c_void_p
L.sdx_kernel_last_error.restype = C.c_char_p
L.sdx_taesd_create.argtypes = [C.c_int, C.c_uint64, C.c_int, C.POINTER(vp)]
L.sdx_taesd_profile.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_double),
                                C.POINTER(C.c_float), C.POINTER(C.c_int)]
imgs = [int(a) for a in sys.argv[1:]] or [1, 8]
h = vp()
assert L.sdx_taesd_create(max(imgs), 77, 0, C.byref(h)) == 0, L.sdx_kernel_last_error()
cap = 256
labels, flops, ms, n = (C.c_char_p * cap)(), (C.c_double * cap)(), (C.c_float * cap)(), C.c_int()
for im in imgs:
    for dec in (0, 1):
        assert L.sdx_taesd_profile(h, dec, im, cap, labels, flops, ms, C.byref(n)) == 0, L.sdx_kernel_last_error()
        acc = collections.OrderedDict()
        for i in range(n.value):
            a = acc.setdefault(labels[i].decode(), [0, 0.0, 0.0])
            a[0] += 1
            a[1] += ms[i]
            a[2] += flops[i]
        tot = sum(v[1] for v in acc.values())
        tf = sum(v[2] for v in acc.values())
        print(f"=== {'decoder' if dec else 'encoder'} x{im} images: {tot:.3f} ms, {n.value} ops, "
              f"{tf / tot / 1e9:.1f} TFLOP/s")
        for lab, (c, t, f) in acc.items():
            print(f"  {t:8.4f} ms {100 * t / tot:5.1f}% x{c:<2d} {f / t / 1e9 if t else 0:7.1f} TF/s  {lab}")
