"""CPU: the results/profile harness reproduces the reference's formats —
the acceptance fixture of criterion 11 (acceptance_main.cpp:440-477) and the
22-column BenchRecord CSV (bench.cpp:28-102)."""
import pytest

from paper_1801_03065_b200 import harness as H


def _rec(problem, algo, t):
    return H.BenchRecord(problem=problem, algorithm=algo, scheme="seq", t_total_ms=t)


def test_profile_fixture_matches_reference_criterion_11(tmp_path):
    rows = [_rec("p1", "A", 10.0), _rec("p2", "A", 10.0), _rec("p3", "A", 10.0),
            _rec("p1", "B", 10.0), _rec("p2", "B", 20.0), _rec("p3", "B", 40.0)]
    inp, out = tmp_path / "in.csv", tmp_path / "out.csv"
    H.write_bench_csv(str(inp), rows)
    assert H.main(["profile", "--in", str(inp), "--out", str(out), "--points", "3"]) == 0
    assert out.read_text() == "x,A,B\n1,3,1\n2,3,2\n4,3,3\n"


def test_csv_roundtrip_and_header(tmp_path):
    r = H.BenchRecord("c2", "auto", "seq", 10, 10, 10, 27, 27, 729, 81, 125, 13, 0.35, 0.55, 1, 5, True,
                      1.5, 2.5, 3.5, 7.5, 0.2)
    p = tmp_path / "r.csv"
    H.write_bench_csv(str(p), [r])
    text = p.read_text().splitlines()
    assert text[0] == H.HEADER
    assert text[1] == ("c2,auto,seq,10,10,10,27,27,729,81,125,13,0.350000,0.550000,1,5,1,1.500000,"
                       "2.500000,3.500000,7.500000,0.200000")
    back = H.read_bench_csv(str(p))[0]
    assert back.flops == 729 and back.reuse and back.t_total_ms == 7.5
    assert (tmp_path / "r.gpu.csv").exists()


def test_profile_needs_two_methods():
    with pytest.raises(ValueError):
        H.compute_profile([_rec("p1", "A", 1.0)], 3)


def test_reference_cli_reads_our_csv(tmp_path, reference):
    """The reference's own read_bench_csv/compute_profile (through its run_cli
    stub binary) consumes the GPU harness CSV."""
    import os
    import subprocess
    rows = [_rec("p1", "A", 10.0), _rec("p2", "A", 10.0), _rec("p3", "A", 10.0),
            _rec("p1", "B", 10.0), _rec("p2", "B", 20.0), _rec("p3", "B", 40.0)]
    inp = tmp_path / "in.csv"
    H.write_bench_csv(str(inp), rows)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "oracle", "_ref", "acceptance_ref")
    if not os.path.exists(exe):
        pytest.skip("reference binaries not built")
    import ctypes
    lib = reference.L
    lib.ref_profile_csv.restype = ctypes.c_int
    lib.ref_profile_csv.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int]
    theirs, ours = tmp_path / "ref_profile.csv", tmp_path / "our_profile.csv"
    assert lib.ref_profile_csv(str(inp).encode(), str(theirs).encode(), 7) == 0
    H.write_profile_csv(str(ours), H.compute_profile(H.read_bench_csv(str(inp)), 7))
    assert ours.read_text() == theirs.read_text()
    del subprocess, exe
