"""Config 4 (R-MAT scale 20, ef 16) end to end on one GPU: symbolic stats vs
SURVEY §8d, numeric timing, row-sampled parity vs the oracle."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))  # repo root
import numpy as np, torch
import paper_1801_03065_b200 as kk
from paper_1801_03065_b200 import generators as G
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
budget = int(float(sys.argv[2]) * 2**30) if len(sys.argv) > 2 else 1 << 30
t = time.time(); a = G.rmat(scale, 16, 1); print("gen", round(time.time() - t, 1), "s nnz", a.nnz(), flush=True)
A = a.to_device()
cfg = kk.SpgemmConfig(pool_budget_bytes=budget)
torch.cuda.synchronize(); t = time.time()
h = kk.symbolic(A, A, cfg); torch.cuda.synchronize(); tsym = time.time() - t
info = h._info()
print(json.dumps({"sym_s": round(tsym, 3), "flops": info.flops.total_flops, "nnz_c": info.nnz_c,
                  "max_row_size": info.max_row_size, "max_row_flops": info.flops.max_row_flops,
                  "cf": info.compression.cf, "cmrf": info.compression.cmrf,
                  "sym_pool_allocs": info.symbolic_stats.pool_allocations}), flush=True)
st = kk.PhaseStats()
t = time.time(); c = kk.numeric(A, A, h, st); torch.cuda.synchronize(); tnum = time.time() - t
print(json.dumps({"num_s": round(tnum, 3), "num_ms_events": st.ms, "pool_allocs": st.pool_allocations,
                  "l2_inserts": st.l2_inserts, "gflops_num": 2 * info.flops.total_flops / tnum / 1e9,
                  "gflops_symnum": 2 * info.flops.total_flops / (tsym + tnum) / 1e9}), flush=True)
# row-sampled parity: every 64th row + the 256 heaviest rows
from oracle.oracle import Oracle
o = Oracle()
ro = h.c_row_offsets
sizes = np.diff(ro)
rows = np.unique(np.concatenate([np.arange(0, a.num_rows, 64), np.argsort(sizes)[-256:]]))
lo, hi = a.row_offsets[rows], a.row_offsets[rows + 1]
sro = np.zeros(len(rows) + 1, np.int64); np.cumsum(hi - lo, out=sro[1:])
idx = np.concatenate([np.arange(l, e) for l, e in zip(lo, hi)])
asamp = kk.CsrMatrix(len(rows), a.num_cols, sro, a.col_indices[idx], a.values[idx], True)
t = time.time(); oro, ocols, ovals = o.multiply(asamp, a); print("oracle sample", round(time.time() - t, 1), "s", flush=True)
ok_struct = np.array_equal(np.diff(oro), sizes[rows])
cols_d = c.col_indices; vals_d = c.values
bad = 0; maxrel = 0.0; exact = True
for q, i in enumerate(rows):
    gs, ge = int(ro[i]), int(ro[i + 1])
    gc = cols_d[gs:ge].cpu().numpy(); gv = vals_d[gs:ge].cpu().numpy()
    oc = ocols[oro[q]:oro[q + 1]]; ov = ovals[oro[q]:oro[q + 1]]
    if not np.array_equal(gc, oc) or not np.array_equal(gv.view(np.int64), ov.view(np.int64)):
        exact = False
        sg = np.argsort(gc); so = np.argsort(oc)
        if not np.array_equal(gc[sg], oc[so]):
            bad += 1; continue
        maxrel = max(maxrel, o.max_rel_error(ov[so], gv[sg]))
print(json.dumps({"sample_rows": len(rows), "structure_equal": bool(ok_struct and bad == 0), "bad_rows": bad,
                  "bitwise_raw_equal": exact, "max_rel": maxrel}), flush=True)
