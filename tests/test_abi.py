"""CPU: the C-ABI library loads, exports every symbol include/kkspgemm.h
declares, its pure-host entry points (resolve_config, flat_position) match the
reference's KATs, and compute entry points fail loudly without a GPU (there is
no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def kk():
    import paper_1801_03065_b200 as kk
    if not os.path.exists(kk.LIB_PATH):
        from paper_1801_03065_b200.build import build_kkspgemm
        build_kkspgemm()
    return kk


def header_symbols():
    with open(os.path.join(ROOT, "include", "kkspgemm.h")) as f:
        text = f.read()
    return set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(spg_[a-z_0-9]+)\s*\(", text, re.M))


def test_every_declared_symbol_is_exported(kk):
    lib = ctypes.CDLL(kk.LIB_PATH)
    declared = header_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(kk.EXPORTED_SYMBOLS)


def test_library_is_sm100a(kk):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", kk.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_resolve_config_kats(kk, kats):
    for c in kats["resolve_config"]["cases"]:
        st = kk.FlopsStats(avg_row_flops=c["avg_row_flops"])
        rep = kk.CompressionReport(applied=c["applied"])
        r = kk.resolve_config(c["phase"], c["k"], st, rep, kk.SpgemmConfig(), c["bound"])
        if "acc" in c:
            assert r.accumulator == c["acc"], c
        if "acc_not" in c:
            assert r.accumulator != c["acc_not"], c
        if "scheme" in c:
            assert r.scheme == c["scheme"], c
        if "effective_k" in c:
            assert r.effective_k == c["effective_k"], c


def test_resolve_config_matches_oracle_grid(kk, oracle):
    for phase in (0, 1):
        for k in (1, 31, 32, 33, 249_999, 250_000, 8_000_000, 7_999_999):
            for avg in (0.0, 255.9, 256.0, 300.0):
                for applied in (False, True):
                    for bound in (0, 1, 100, 10**9):
                        r = kk.resolve_config(phase, k, kk.FlopsStats(avg_row_flops=avg),
                                              kk.CompressionReport(applied=applied), kk.SpgemmConfig(), bound)
                        o = oracle.resolve_config(phase, k, avg, applied, bound=bound)
                        assert (r.accumulator, r.scheme, r.l1_capacity, r.effective_k, r.l2_capacity) == (
                            o["accumulator"], o["scheme"], o["l1_capacity"], o["effective_k"],
                            o["l2_capacity"])


def test_flat_position_kats(kk, kats):
    g = kats["flat_position"]
    for t, seg, off in g["cases"]:
        assert kk.flat_position(g["prefix"], t) == (seg, off)


def test_compute_without_gpu_fails_loudly(kk):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np
    a = kk.CsrMatrix(1, 1, np.array([0, 1], np.int64), np.array([0], np.int32), np.array([1.0]), True)
    with pytest.raises(Exception):
        kk.symbolic(a, a)
