"""Randomised parity fuzzing of the GPU engine against the oracle.

Each case draws shapes, densities, row-length skew, sortedness, a config
(accumulator, scheme, l1_capacity, compression, sort_output) and a path
(multiply, reuse passes incl. slot replay, row ranges, row-block views, host
multiply) and checks C against the C oracle bit for bit (raw order when
the reference's raw order is defined, sorted otherwise).

    python tests/tools/fuzz.py [seconds] [seed]

Test infrastructure: the oracle is the checker.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))  # repo root
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # tests/ (conftest helpers)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_03065_b200 as kk  # noqa: E402
from conftest import random_csr  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_1801_03065_b200 import host  # noqa: E402


def skewed_csr(rng, m, n, density, shuffle):
    """random_csr with a few heavy rows appended."""
    a = random_csr(rng, m, n, density, shuffle=shuffle)
    if m == 0 or n == 0 or rng.random() < 0.5:
        return a
    heavy = rng.choice(m, max(1, m // 50), replace=False)
    rows = []
    for i in range(m):
        lo, hi = a.row_offsets[i], a.row_offsets[i + 1]
        cols = list(a.col_indices[lo:hi])
        vals = list(a.values[lo:hi])
        if i in heavy:
            extra = rng.choice(n, min(n, int(rng.integers(n // 4 + 1, n + 1))), replace=False)
            have = set(cols)
            for c in extra:
                if c not in have:
                    cols.append(int(c))
                    vals.append(float(rng.standard_normal()))
        order = np.arange(len(cols)) if shuffle else np.argsort(cols, kind="stable")
        rows.append(([cols[q] for q in order], [vals[q] for q in order]))
    ro = np.zeros(m + 1, np.int64)
    ro[1:] = np.cumsum([len(r[0]) for r in rows])
    ci = np.array([c for r in rows for c in r[0]], np.int32)
    v = np.array([x for r in rows for x in r[1]], np.float64)
    return kk.CsrMatrix(m, n, ro, ci, v, not shuffle)


def wide_csr(rng, m, n, density, shuffle):
    """Random CSR over many columns (sampling with replacement, duplicates
    dropped) — random_csr's per-row permutation is too slow at n ~ 1e5."""
    cnt = rng.binomial(n, density, m) if n > 0 else np.zeros(m, np.int64)
    key = np.sort(np.repeat(np.arange(m, dtype=np.int64), cnt) * max(n, 1)
                  + rng.integers(0, max(n, 1), int(cnt.sum())))
    key = key[np.concatenate(([True], key[1:] != key[:-1]))] if len(key) else key
    rows, ci = key // max(n, 1), (key % max(n, 1)).astype(np.int32)
    ro = np.zeros(m + 1, np.int64)
    ro[1:] = np.cumsum(np.bincount(rows, minlength=m))
    if shuffle:
        ci = ci[np.argsort(rows + rng.random(len(ci)))]
    return kk.CsrMatrix(m, n, ro, ci, rng.uniform(-1, 1, len(ci)), not shuffle)


def check(o, a, b, c, raw):
    ro = o.symbolic_row_offsets(a, b)
    assert np.array_equal(c.row_offsets, ro), "row offsets"
    cols, vals = o.numeric(a, b, ro)
    sc, sv = o.sort_rows(ro, cols, vals)
    gc, gv = o.sort_rows(ro, c.col_indices, c.values)
    assert np.array_equal(sc, gc), "sorted columns"
    assert np.array_equal(sv.view(np.int64), gv.view(np.int64)), "sorted value bits"
    if raw:
        assert np.array_equal(c.col_indices, cols), "raw column order"


def one_case(rng, o):
    u = rng.random()
    if u < 0.06:
        # long A rows over wide B: many column slabs per row, replans and
        # table-overflow aborts in the column-slab kernel
        m, n, k = int(rng.integers(1, 12)), int(rng.integers(1000, 4000)), int(rng.integers(20000, 200000))
        da, db = float(rng.choice([0.1, 0.3, 0.6])), float(rng.choice([0.002, 0.005, 0.01]))
    elif u < 0.16:
        # a few rows beyond the warp tables (heavy CTA path / L2 pool)
        m, n, k = int(rng.integers(1, 48)), int(rng.integers(500, 3000)), int(rng.integers(3000, 30000))
        da, db = float(rng.choice([0.02, 0.08])), float(rng.choice([0.01, 0.03]))
    else:
        m, n, k = (int(x) for x in rng.integers(0, 400, 3))
        da = float(rng.choice([0.005, 0.02, 0.08, 0.2]))
        db = float(rng.choice([0.005, 0.02, 0.08, 0.2]))
    shuffle = bool(rng.random() < 0.3)
    if u < 0.06:
        a = wide_csr(rng, m, n, da, shuffle)
        b = wide_csr(rng, n, k, db, shuffle)
    else:
        a = skewed_csr(rng, m, n, da, shuffle)
        b = skewed_csr(rng, n, k, db, shuffle)
    acc = int(rng.choice([0, 0, 0, 1, 2, 3]))
    cfg = kk.SpgemmConfig(accumulator=acc, scheme=int(rng.integers(0, 2)),
                          l1_capacity=int(rng.choice([0, 0, 0, 1, 16])) if acc != 3 else 0,
                          compression=int(rng.integers(0, 3)), sort_output=bool(rng.random() < 0.2))
    path = rng.choice(["multiply", "reuse", "rows", "view", "host"])
    raw = not cfg.sort_output
    if path == "multiply":
        c = kk.multiply(a, b, cfg).c.to_host()
        # heavy rows of the Auto plan come out in their own order
        check(o, a, b, c, raw and acc != 0)
    elif path == "reuse":
        h = kk.symbolic(a, b, cfg)
        for p in range(4):
            ap = kk.CsrMatrix(a.num_rows, a.num_cols, a.row_offsets, a.col_indices,
                              a.values * (1.0 + 0.25 * p), a.sorted_rows)
            c = kk.numeric(ap, b, h, kk.PhaseStats()).to_host()
            check(o, ap, b, c, raw and acc != 0)
    elif path == "rows":
        dA, dB = a.to_device(), b.to_device()
        h = kk.symbolic(dA, dB, cfg)
        nnz = h.nnz_c()
        cols = torch.full((max(nnz, 1),), -5, dtype=torch.int32, device="cuda")
        vals = torch.zeros(max(nnz, 1), dtype=torch.float64, device="cuda")
        cuts = sorted(set([0, m] + [int(x) for x in rng.integers(0, m + 1, 3)]))
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            kk.numeric_rows(dA, dB, h, r0, r1, cols, vals)
        if cfg.sort_output is False:
            c = kk.CsrMatrix(m, k, h.c_row_offsets, cols.cpu().numpy()[:nnz], vals.cpu().numpy()[:nnz])
            check(o, a, b, c, False)
    elif path == "view":
        if m < 2:
            return path
        lo = int(rng.integers(0, m))
        hi = int(rng.integers(lo, m + 1))
        dA, dB = a.to_device(), b.to_device()
        c = kk.multiply(dA.row_block(lo, hi), dB, cfg).c.to_host()
        sub = kk.CsrMatrix(hi - lo, n, a.row_offsets[lo:hi + 1] - a.row_offsets[lo],
                           a.col_indices[a.row_offsets[lo]:a.row_offsets[hi]],
                           a.values[a.row_offsets[lo]:a.row_offsets[hi]], a.sorted_rows)
        check(o, sub, b, c, raw and acc != 0)
    else:
        r = host.multiply_host(host.PinnedCsr.from_csr(a), host.PinnedCsr.from_csr(b), cfg,
                               blocks=int(rng.integers(1, 4)))
        check(o, a, b, r.c, False)
    return path


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    o = Oracle()
    t0 = time.time()
    n = 0
    paths = {}
    while time.time() - t0 < secs:
        state = rng.bit_generator.state
        try:
            p = one_case(rng, o)
        except Exception as e:  # report the reproducible case and stop
            print(f"FAIL after {n} cases (seed {seed}, rng state {state['state']['state']}): {e!r}")
            raise
        paths[p] = paths.get(p, 0) + 1
        n += 1
    print(f"fuzz ok: {n} cases in {time.time() - t0:.0f} s, paths {paths}")


if __name__ == "__main__":
    main()
