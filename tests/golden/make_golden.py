"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED
reference library (oracle/_ref/libspgemm_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py

Outputs (committed; /root/reference is absent on the GPU box):
  reference_kats.json   known-answer tests transcribed from the reference's own
                        test suites (file:line in each entry) and re-checked here
                        against the reference library
  instances.npz         randomized instances (the reference's own fixture
                        generators test_util.hpp) with the reference's raw
                        symbolic/numeric output (row offsets, first-touch
                        columns, values bit for bit) and handle statistics
  configs.json          BASELINE configs at reduced scale: the reference's
                        handle statistics and SHA-256 digests of its raw output
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_1801_03065_b200 import generators as G  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def kats(ref: Reference) -> dict:
    out = {}
    # engine_test.cpp:46-64, oracle_test.cpp:32-48
    a = ref.build_csr(3, 3, [(0, 0, 1), (0, 2, 2), (1, 1, 3), (2, 0, 4), (2, 2, 5)])
    b = ref.build_csr(3, 3, [(0, 0, 1), (0, 1, 1), (1, 1, 2), (2, 2, 3)])
    h = ref.symbolic(a, b)
    cols, vals, _ = h.numeric()
    out["hand_3x3"] = {
        "cite": "tests/engine_test.cpp:46-64, tests/oracle_test.cpp:32-48",
        "a": [(0, 0, 1), (0, 2, 2), (1, 1, 3), (2, 0, 4), (2, 2, 5)],
        "b": [(0, 0, 1), (0, 1, 1), (1, 1, 2), (2, 2, 3)],
        "row_offsets": [0, 3, 4, 7],
        "canonical": [[[0, 1.0], [1, 1.0], [2, 6.0]], [[1, 6.0]], [[0, 4.0], [1, 4.0], [2, 15.0]]],
        "reference_raw_cols": cols.tolist(), "reference_raw_vals": vals.tolist(),
    }
    assert h.row_offsets().tolist() == [0, 3, 4, 7]
    # matrix_test.cpp:99-109
    a = ref.build_csr(2, 2, [(0, 0, 1), (0, 1, 1)])
    b = ref.build_csr(2, 4, [(0, 0, 1), (0, 1, 1), (1, 0, 1), (1, 2, 1), (1, 3, 1)])
    per, tot, mx = ref.flops_stats(a, b)
    assert per.tolist() == [5, 0] and tot == 5 and mx == 5
    out["flops_5_0"] = {"cite": "tests/matrix_test.cpp:99-109",
                        "a": [(0, 0, 1), (0, 1, 1)], "a_shape": [2, 2],
                        "b": [(0, 0, 1), (0, 1, 1), (1, 0, 1), (1, 2, 1), (1, 3, 1)], "b_shape": [2, 4],
                        "per_row_flops": [5, 0], "total": 5, "max": 5}
    # compression_test.cpp:12-33
    out["compress_prefix"] = {"cite": "tests/compression_test.cpp:12-21",
                              "cols": list(range(10)), "k": 40, "pairs": [[0, 0x3FF]]}
    out["compress_split"] = {"cite": "tests/compression_test.cpp:23-33",
                             "cols": [1, 3, 33], "k": 64, "pairs": [[0, 0b1010], [1, 0b10]]}
    # compression_test.cpp:101-132 (gate boundary)
    out["gate_exact_15"] = {"cite": "tests/compression_test.cpp:101-117",
                            "b_cols": sorted([w * 32 for w in range(17)] + [1, 2, 3]), "k": 17 * 32,
                            "flops": 20, "compressed_flops": 17, "applied": False}
    out["gate_16_of_20"] = {"cite": "tests/compression_test.cpp:119-132",
                            "b_cols": sorted([w * 32 for w in range(16)] + [1, 2, 3, 4]), "k": 16 * 32,
                            "flops": 20, "compressed_flops": 16, "applied": True}
    for key in ("gate_exact_15", "gate_16_of_20"):
        g = out[key]
        bb = ref.build_csr(1, g["k"], [(0, c, 1.0) for c in g["b_cols"]])
        aa = ref.build_csr(1, 1, [(0, 0, 1.0)])
        hh = ref.symbolic(aa, bb)
        info = hh.info()
        assert info["compressed_flops"] == g["compressed_flops"] and bool(info["applied"]) == g["applied"]
    # engine_test.cpp:147-156
    out["flat_position"] = {"cite": "tests/engine_test.cpp:147-156", "prefix": [0, 3, 8],
                            "cases": [[5, 1, 2], [0, 0, 0], [7, 1, 4]]}
    # engine_test.cpp:282-326, acceptance_main.cpp:303-331
    out["resolve_config"] = {"cite": "tests/engine_test.cpp:282-326", "cases": [
        {"phase": 1, "k": 10000, "avg_row_flops": 50.0, "applied": False, "bound": 100, "acc": 3},
        {"phase": 1, "k": 1000000, "avg_row_flops": 50.0, "applied": False, "bound": 100, "acc": 1, "scheme": 0},
        {"phase": 1, "k": 1000000, "avg_row_flops": 500.0, "applied": False, "bound": 100, "acc": 2, "scheme": 1},
        {"phase": 0, "k": 1000000, "avg_row_flops": 500.0, "applied": True, "bound": 100, "acc": 3, "effective_k": 31250},
        {"phase": 1, "k": 1000000, "avg_row_flops": 500.0, "applied": True, "bound": 100, "acc": 2},
        {"phase": 1, "k": 250000, "avg_row_flops": 50.0, "applied": False, "bound": 10, "acc_not": 3},
        {"phase": 1, "k": 1000000, "avg_row_flops": 256.0, "applied": False, "bound": 10, "acc": 2},
    ]}
    # engine_test.cpp:243-250
    out["cancellation"] = {"cite": "tests/engine_test.cpp:243-250",
                           "a": [(0, 0, 1.0), (0, 1, -1.0)], "a_shape": [1, 2],
                           "b": [(0, 0, 5.0), (1, 0, 5.0)], "b_shape": [2, 1], "nnz_c": 1, "value": 0.0}
    # acceptance_main.cpp:276-298 / PAPER.md:981,993 (data files absent: kept for the record)
    out["paper_statistics"] = {"cite": "tests/acceptance_main.cpp:276-298",
                               "amazon0302": {"flops": 6021131, "nnz_c": 3896236, "max_row_flops": 25,
                                              "max_row_size": 25, "cf": 0.71, "cmrf": 1.00},
                               "web-Google": {"flops": 60687836, "nnz_c": 29710164, "cf": 1.00},
                               "status": "SKIP: matrices not available offline"}
    return out


def instances(ref: Reference) -> dict:
    arrays = {}
    meta = []
    rng = ref.rng(0x5EED)
    kinds = []
    for it in range(24):
        m, n, k = [int(x) for x in np.random.RandomState(1000 + it).randint(1, 160, 3)]
        if it % 3 == 0:
            a = ref.shuffle_rows(ref.random_csr(rng, m, n, 0.08), it)
            b = ref.shuffle_rows(ref.random_csr(rng, n, k, 0.08), it + 1)
            kinds.append("random_shuffled")
        else:
            ta = max(1, min(n, 3 + it % 7))
            tb = max(1, min(k, 2 + it % 5))
            a = ref.synthetic_by_index(it, m, n, ta, 500 + it)
            b = ref.synthetic_by_index(it + 1, n, k, tb, 900 + it)
            kinds.append("synthetic")
        h = ref.symbolic(a, b)
        cols, vals, _ = h.numeric()
        info = h.info()
        p = f"i{it}_"
        for name, mat in (("a", a), ("b", b)):
            arrays[p + name + "_shape"] = np.array([mat.num_rows, mat.num_cols], np.int64)
            arrays[p + name + "_ro"] = mat.row_offsets
            arrays[p + name + "_ci"] = mat.col_indices
            arrays[p + name + "_v"] = mat.values
        arrays[p + "c_ro"] = h.row_offsets()
        arrays[p + "c_ci"] = cols
        arrays[p + "c_v"] = vals
        arrays[p + "per_row_flops"] = h.per_row_flops()
        meta.append({k2: info[k2] for k2 in ("total_flops", "max_row_flops", "compressed_flops",
                                               "compressed_max_row_flops", "applied", "max_row_size",
                                               "nnz_c", "sym_acc", "sym_scheme", "sym_effk", "num_acc",
                                               "num_scheme", "num_l2")})
    arrays["meta"] = np.frombuffer(json.dumps({"instances": meta, "kinds": kinds}).encode(), np.uint8)
    return arrays


def configs(ref: Reference) -> dict:
    out = {}
    cases = {
        "c1_2d_n100": lambda: (G.laplace2d(100), None),
        "c2_3d_n16": lambda: (G.laplace3d(16), None),
        "c3_ap_n12": lambda: (G.laplace3d(12), G.aggregation(12)),
        "c4_rmat_s10": lambda: (G.rmat(10, 16, 1), None),
        "c5_3d_n20": lambda: (G.laplace3d(20), None),
    }
    for name, make in cases.items():
        a, b = make()
        b = a if b is None else b
        h = ref.symbolic(a, b, worker_count=4)
        cols, vals, _ = h.numeric()
        info = h.info()
        entry = {k2: info[k2] for k2 in ("m", "n", "k", "nnz_a", "nnz_b", "nnz_c", "total_flops",
                                         "max_row_flops", "compressed_flops", "compressed_max_row_flops",
                                         "applied", "max_row_size", "sym_acc", "sym_effk", "num_acc",
                                         "num_scheme")}
        entry["cf"] = info["cf"]
        entry["cmrf"] = info["cmrf"]
        entry["inputs_sha256"] = digest(a.row_offsets, a.col_indices, a.values, b.row_offsets,
                                        b.col_indices, b.values)
        entry["row_offsets_sha256"] = digest(h.row_offsets())
        entry["raw_cols_sha256"] = digest(cols)
        entry["raw_vals_sha256"] = digest(vals)
        out[name] = entry
        if name == "c3_ap_n12":  # the chained R*(AP) as well
            r = G.transpose(b)
            from paper_1801_03065_b200 import CsrMatrix
            ap = CsrMatrix(a.num_rows, b.num_cols, h.row_offsets(), cols, vals, False)
            h2 = ref.symbolic(r, ap, worker_count=4)
            c2, v2, _ = h2.numeric()
            i2 = h2.info()
            out["c3_rap_n12"] = {"nnz_c": i2["nnz_c"], "total_flops": i2["total_flops"],
                                 "applied": i2["applied"], "cf": i2["cf"],
                                 "row_offsets_sha256": digest(h2.row_offsets()),
                                 "raw_cols_sha256": digest(c2), "raw_vals_sha256": digest(v2)}
    return out


def main():
    ref = Reference()
    with open(os.path.join(HERE, "reference_kats.json"), "w") as f:
        json.dump(kats(ref), f, indent=1)
    np.savez_compressed(os.path.join(HERE, "instances.npz"), **instances(ref))
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(configs(ref), f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
