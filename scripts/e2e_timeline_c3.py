"""Timeline of the c3 host-memory triple product (two host.multiply_host
calls, A*P then R*(AP)): event marks of both calls and host wall times."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_03065_b200 as kk  # noqa: E402
from bench import workload  # noqa: E402
from paper_1801_03065_b200 import generators as G  # noqa: E402
from paper_1801_03065_b200 import host  # noqa: E402

mats, wl = workload(3, 1.0, G)
a, p = mats["A"], mats["P"]
r = kk.transpose(p.to_device()).to_host()
pa, pp, pr = (host.PinnedCsr.from_csr(x) for x in (a, p, r))
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tl1, tl2 = [], []
    r1 = host.multiply_host(pa, pp, timeline=tl1)
    t1 = time.perf_counter()
    o_ro, o_ci, o_v = r1._keep
    n1 = r1.c.nnz()
    ap = host.PinnedCsr(a.num_rows, p.num_cols, o_ro[:a.num_rows + 1], o_ci[:n1], o_v[:n1], False)
    r2 = host.multiply_host(pr, ap, timeline=tl2)
    t2 = time.perf_counter()
    print(it, f"A*P {1e3 * (t1 - t0):.1f} ms, R*AP {1e3 * (t2 - t1):.1f} ms")
    for tl in (tl1, tl2):
        e0 = tl[0][1]
        print("   ", [(lbl, round(e0.elapsed_time(e), 2)) for lbl, e in tl])
