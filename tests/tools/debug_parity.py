"""Debug helper: which (phase, accumulator, scheme, compression) disagrees with the oracle."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))  # repo root
import paper_1801_03065_b200 as kk
from paper_1801_03065_b200 import generators as G
from oracle.oracle import Oracle
o = Oracle()
a = G.laplace3d(6)
ro = o.symbolic_row_offsets(a, a)
print("oracle nnz", ro[-1], "flops", o.flops_stats(a, a)[1])
for comp in (1, 2):
    for acc in (1, 2, 3):
        for sch in (0, 1):
            cfg = kk.SpgemmConfig(accumulator=acc, scheme=sch, compression=comp)
            try:
                h = kk.symbolic(a, a, cfg)
                g = h.c_row_offsets
                sz, osz = np.diff(g), np.diff(ro)
                bad = np.nonzero(sz != osz)[0]
                print(f"comp={comp} acc={acc} sch={sch}: nnz {g[-1]} bad rows {len(bad)}",
                      [(int(i), int(sz[i]), int(osz[i])) for i in bad[:5]])
                if len(bad) == 0:
                    c = kk.numeric(a, a, h, kk.PhaseStats()).to_host()
                    cols, vals = o.numeric(a, a, ro)
                    print("   numeric cols eq", np.array_equal(c.col_indices, cols),
                          "vals eq", np.array_equal(c.values, vals))
            except Exception as e:
                print(f"comp={comp} acc={acc} sch={sch}: EXC {e}")
