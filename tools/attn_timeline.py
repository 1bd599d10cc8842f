"""Phase timeline of one attention CTA (clock64 stamps, sdx_kernel_attention_debug):
per KV block, per softmax warp: wait-S, TMEM load, max, exponentials; per tile, when the
MMA warp saw P and issued PV + the next S.

    python tools/attn_timeline.py [imgs T heads]
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_12491_b200 import _lib  # noqa: E402

L = _lib.lib
vp, i64 = C.c_void_p, C.c_int64
L.sdx_kernel_attention.argtypes = [vp, i64, i64, C.c_int, vp, i64, i64, C.c_int, C.c_int, vp, i64, C.c_int, C.c_int,
                                   C.c_int, C.c_int, C.c_int, vp, C.c_float, vp]
L.sdx_kernel_attention_debug.argtypes = [vp]
imgs, T, heads = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4, 4096, 5)
Cd = heads * 64
qkv = torch.randn(imgs * T, 3 * Cd, device="cuda").bfloat16()
out = torch.zeros(imgs * T, Cd, device="cuda", dtype=torch.bfloat16)
dbg = torch.zeros(11 * 64 * 8, dtype=torch.int64, device="cuda")
run = lambda: L.sdx_kernel_attention(qkv.data_ptr(), imgs * T, 3 * Cd, 0, qkv.data_ptr(), imgs * T, 3 * Cd, Cd,  # noqa
                                     2 * Cd, out.data_ptr(), Cd, imgs, heads, T, T, T, None, 0.125, None)
run()
torch.cuda.synchronize()
L.sdx_kernel_attention_debug(dbg.data_ptr())
run()
torch.cuda.synchronize()
L.sdx_kernel_attention_debug(None)
d = dbg.view(11, 64, 8).cpu().numpy()
t0 = d[0, 0, 7]
nkv = min(64, (T + 127) // 128)
print("block | warp2(t0): wait-S  ld  max+pvwait  exp | warp6(t1): same | mma: P seen, PV issue time, next S issued")
prev = [None, None]
for j in range(nkv):
    row = f"{j:3d} |"
    for w in (3, 7):
        e = d[w, j]
        row += f" start {e[0] - t0:7d} wS {e[1] - e[0]:5d} ld {e[2] - e[1]:4d} mx {e[3] - e[2]:4d} ex {e[4] - e[3]:5d} |"
    m, m1 = d[1, j], d[2, j]
    row += (f" P0 {m[0] - t0:7d} pv {m[2] - m[0]:4d} S0(j+1) {m[1] - t0:7d}"
            f" P1 {m1[0] - t0:7d} pv {m1[2] - m1[0]:4d} S1(j+1) {m1[1] - t0:7d}")
    print(row)
tot = d[3, nkv - 1, 4] - d[3, 0, 0]
print(f"tile0 cycles for {nkv} blocks: {tot}, per block {tot / nkv:.0f}")
print("P-ready skew across the 4 warps of each tile (exp end, relative to warp 3 / 7):")
for j in range(min(nkv, 8)):
    e0 = [int(d[w, j, 4] - d[3, j, 4]) for w in (3, 4, 5, 6)]
    e1 = [int(d[w, j, 4] - d[7, j, 4]) for w in (7, 8, 9, 10)]
    print(f"{j:3d} tile0 {e0}  tile1 {e1}  | MMA0 saw P {int(d[1, j, 0] - d[3, j, 4])} after warp3")
