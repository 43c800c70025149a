"""Phase profile of the column-slab heavy kernel (build with -DKK_SLAB_PROF).
Usage: python scripts/slab_prof.py [scale]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_03065_b200 as kk  # noqa: E402
from paper_1801_03065_b200 import generators as G  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
a = G.rmat(scale, 16, 1)
A = a.to_device()
h = kk.symbolic(A, A)
L = kk.lib()
f = L.spg_debug_slab_prof
f.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 64)()
c = kk.numeric(A, A, h)
torch.cuda.synchronize()
f(None, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
kk.numeric(A, A, h, out=(c.col_indices, c.values))
e1.record()
torch.cuda.synchronize()
f(buf, 0)
names = ["cursor_init_cyc", "plan_cyc", "fold_cyc", "emit_cyc", "", "", "", "",
         "slabs", "products", "replans", "aborts", "replans_narrower", "replans_wider", "runs_planned",
         "entries_planned"]
print(f"s{scale} numeric {e0.elapsed_time(e1):.2f} ms heavy_path={h.heavy_path}")
for n, v in zip(names, buf):
    if n:
        print(f"  {n:16s} {v:>18,d}")
print("  by A-row length class (item cycles, outputs, items):")
tot = sum(buf[16:32]) or 1
for c in range(16):
    if buf[48 + c]:
        print(f"   d<=2^{c:2d}: {100 * buf[16 + c] / tot:5.1f}% cycles  outputs {buf[32 + c]:>14,d}  items {buf[48 + c]:>8,d}")
