"""Per-op device times of the UNet forward (CUDA events around every op), with
each GEMM / attention op's shape and achieved TFLOP/s.

    python tools/prof_ops.py [rows] [iters]
"""
import collections
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2312_12491_b200 import _lib  # noqa: E402

L = _lib.lib
L.sdx_kernel_last_error.restype = C.c_char_p
vp = C.c_void_p
L.sdx_unet_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.c_uint64, C.c_int, C.POINTER(vp)]
L.sdx_unet_forward.argtypes = [vp, vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), vp, vp]
L.sdx_unet_profile_detail.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_double),
                                      C.POINTER(C.c_float), C.POINTER(C.c_int)]
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
taus = (C.c_int * 4)(999, 749, 499, 249)
h = vp()
assert L.sdx_unet_create(rows, taus, 4, 1234, 0, C.byref(h)) == 0
steps = (C.c_int * rows)(*[i % 4 for i in range(rows)])
prompts = (C.c_int * rows)(*[0] * rows)
for _ in range(3):
    assert L.sdx_unet_forward(h, None, rows, steps, prompts, None, None) == 0
cap = 4096
labels = (C.c_char_p * cap)()
flops = (C.c_double * cap)()
ms = (C.c_float * cap)()
n = C.c_int()
acc = collections.defaultdict(lambda: [0, 0.0, 0.0])  # count, ms, flops
kind_acc = collections.defaultdict(lambda: [0.0, 0.0])
for _ in range(iters):
    rc = L.sdx_unet_profile_detail(h, rows, cap, labels, flops, ms, C.byref(n))
    assert rc == 0, (rc, L.sdx_kernel_last_error())
    for i in range(n.value):
        lab = labels[i].decode()
        a = acc[lab]
        a[0] += 1
        a[1] += ms[i]
        a[2] += flops[i]
        k = kind_acc[lab.split(" ")[0]]
        k[0] += ms[i]
        k[1] += flops[i]
tot = sum(v[1] for v in acc.values()) / iters
print(f"UNet forward, {rows} rows: {tot:.3f} ms per forward ({n.value} ops)")
print("\nby kind:")
for k, (t, f) in sorted(kind_acc.items(), key=lambda kv: -kv[1][0]):
    tf = f / (t * 1e-3) / 1e12 if f else 0.0
    print(f"  {k:16s} {t / iters:8.3f} ms {100 * t / iters / tot:5.1f}%  {tf:7.1f} TFLOP/s")
print("\nby op shape (per forward):")
for lab, (c, t, f) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    tf = f / (t * 1e-3) / 1e12 if f else 0.0
    print(f"  {t / iters:8.3f} ms {100 * t / iters / tot:5.1f}% x{c // iters:<3d} {tf:7.1f} TF/s  {lab}")
