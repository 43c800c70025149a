"""CPU: pin the oracle (C restatement) before trusting it.

* against the reference's own known-answer tests (tests/golden/reference_kats.json,
  each entry cites the reference test file:line it transcribes),
* against the reference library itself (oracle/_ref, compiled from
  /root/reference/proj/src) bit for bit on randomized instances, including the
  raw first-touch column order,
* against the committed golden fixtures (tests/golden/instances.npz,
  configs.json) that the reference produced.
"""
import hashlib

import numpy as np
import pytest

from conftest import csr_from_triplets, load_instances


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_hand_3x3(oracle, kats):
    k = kats["hand_3x3"]
    a = csr_from_triplets(3, 3, k["a"])
    b = csr_from_triplets(3, 3, k["b"])
    ro, cols, vals = oracle.multiply(a, b)
    assert ro.tolist() == k["row_offsets"]
    assert cols.tolist() == k["reference_raw_cols"]
    assert vals.tolist() == k["reference_raw_vals"]
    sc, sv = oracle.sort_rows(ro, cols, vals)
    canon = [[[int(c), float(v)] for c, v in zip(sc[ro[i]:ro[i + 1]], sv[ro[i]:ro[i + 1]])] for i in range(3)]
    assert canon == k["canonical"]


def test_flops_golden(oracle, kats):
    k = kats["flops_5_0"]
    a = csr_from_triplets(*k["a_shape"], k["a"])
    b = csr_from_triplets(*k["b_shape"], k["b"])
    per, tot, mx = oracle.flops_stats(a, b)
    assert per.tolist() == k["per_row_flops"] and tot == k["total"] and mx == k["max"]


@pytest.mark.parametrize("name", ["gate_exact_15", "gate_16_of_20"])
def test_gate_boundary(oracle, kats, name):
    g = kats[name]
    b = csr_from_triplets(1, g["k"], [(0, c, 1.0) for c in g["b_cols"]])
    a = csr_from_triplets(1, 1, [(0, 0, 1.0)])
    d = oracle.decide_compression(a, b)
    assert d["compressed_flops"] == g["compressed_flops"]
    assert d["applied"] == g["applied"]


def test_compressed_sizes_golden(oracle, kats):
    for name in ("compress_prefix", "compress_split"):
        g = kats[name]
        b = csr_from_triplets(1, g["k"], [(0, c, 1.0) for c in g["cols"]])
        assert oracle.compressed_row_sizes(b).tolist() == [len(g["pairs"])]


def test_resolve_config_golden(oracle, kats):
    for c in kats["resolve_config"]["cases"]:
        r = oracle.resolve_config(c["phase"], c["k"], c["avg_row_flops"], c["applied"], bound=c["bound"])
        if "acc" in c:
            assert r["accumulator"] == c["acc"], c
        if "acc_not" in c:
            assert r["accumulator"] != c["acc_not"], c
        if "scheme" in c:
            assert r["scheme"] == c["scheme"], c
        if "effective_k" in c:
            assert r["effective_k"] == c["effective_k"], c


def test_cancellation_kept(oracle, kats):
    k = kats["cancellation"]
    a = csr_from_triplets(*k["a_shape"], k["a"])
    b = csr_from_triplets(*k["b_shape"], k["b"])
    ro, cols, vals = oracle.multiply(a, b)
    assert ro[-1] == k["nnz_c"] and vals.tolist() == [k["value"]]


def test_golden_instances(oracle):
    for inst in load_instances():
        a, b = inst["a"], inst["b"]
        per, tot, mx = oracle.flops_stats(a, b)
        assert np.array_equal(per, inst["per_row_flops"])
        assert tot == inst["meta"]["total_flops"] and mx == inst["meta"]["max_row_flops"]
        d = oracle.decide_compression(a, b)
        assert d["compressed_flops"] == inst["meta"]["compressed_flops"]
        assert d["applied"] == bool(inst["meta"]["applied"])
        ro = oracle.symbolic_row_offsets(a, b)
        assert np.array_equal(ro, inst["c_ro"])
        cols, vals = oracle.numeric(a, b, ro)
        assert np.array_equal(cols, inst["c_ci"])
        assert np.array_equal(vals.view(np.int64), inst["c_v"].view(np.int64))


def test_golden_configs(oracle, config_golden):
    from paper_1801_03065_b200 import generators as G
    cases = {"c1_2d_n100": (G.laplace2d(100), None), "c2_3d_n16": (G.laplace3d(16), None),
             "c3_ap_n12": (G.laplace3d(12), G.aggregation(12)), "c4_rmat_s10": (G.rmat(10, 16, 1), None),
             "c5_3d_n20": (G.laplace3d(20), None)}
    for name, (a, b) in cases.items():
        b = a if b is None else b
        g = config_golden[name]
        assert digest(a.row_offsets, a.col_indices, a.values, b.row_offsets, b.col_indices,
                      b.values) == g["inputs_sha256"], name
        _, tot, mx = oracle.flops_stats(a, b)
        assert (tot, mx) == (g["total_flops"], g["max_row_flops"])
        d = oracle.decide_compression(a, b)
        assert d["compressed_flops"] == g["compressed_flops"] and d["applied"] == bool(g["applied"])
        ro, cols, vals = oracle.multiply(a, b)
        assert digest(ro) == g["row_offsets_sha256"], name
        assert digest(cols) == g["raw_cols_sha256"], name
        assert digest(vals) == g["raw_vals_sha256"], name


def test_oracle_vs_reference_library(oracle, reference):
    """Bitwise agreement with the compiled reference over accumulators x schemes."""
    rng = reference.rng(53)
    rs = np.random.RandomState(7)
    for it in range(16):
        m, n, k = (int(x) for x in rs.randint(1, 120, 3))
        a = reference.shuffle_rows(reference.random_csr(rng, m, n, 0.1), it)
        b = reference.shuffle_rows(reference.random_csr(rng, n, k, 0.1), it + 1)
        ro = oracle.symbolic_row_offsets(a, b)
        cols, vals = oracle.numeric(a, b, ro)
        for acc in (1, 2, 3):
            for scheme in (0, 1):
                h = reference.symbolic(a, b, accumulator=acc, scheme=scheme, worker_count=4)
                assert np.array_equal(h.row_offsets(), ro)
                rc, rv, _ = h.numeric()
                assert np.array_equal(rc, cols)
                assert np.array_equal(rv.view(np.int64), vals.view(np.int64))


def test_generators_match_survey_counts(oracle):
    """SURVEY.md §8d closed forms: nnzA=(3n-2)^3, flops=(9n-10)^3, nnzC=(5n-6)^3."""
    from paper_1801_03065_b200 import generators as G
    for n in (5, 9, 14):
        a = G.laplace3d(n)
        assert a.nnz() == (3 * n - 2) ** 3
        _, tot, _ = oracle.flops_stats(a, a)
        assert tot == (9 * n - 10) ** 3
        assert oracle.symbolic_row_offsets(a, a)[-1] == (5 * n - 6) ** 3
    a = G.laplace2d(50)
    assert a.nnz() == 5 * 50 * 50 - 4 * 50
