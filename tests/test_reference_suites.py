"""The reference's OWN unit and acceptance suites (proj/tests/*.cpp, compiled
unmodified by oracle/Makefile) run twice:

* against the reference engine (CPU) — validates the doctest stand-in and the
  run_cli stub: 85 cases / 38,089 assertions, acceptance criteria 1-5, 7-11;
* against the GPU engine through the engine.hpp shim
  (paper_1801_03065_b200/csrc/engine_shim.cpp) — the drop-in test.

The binaries are built where /root/reference exists (this container) and travel
to the GPU box as build outputs; the tests skip when they were not built.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def _bin(name):
    p = os.path.join(REF, name)
    if not os.path.exists(p):
        if os.path.isdir("/root/reference/proj/src"):
            subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "reftests", "kktests"],
                           check=True)
        else:
            pytest.skip(f"{name} not built (needs /root/reference at build time)")
    return p


def _run(path, timeout):
    try:  # hand device memory cached by earlier tests in this process back
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
    except Exception:
        pass
    r = subprocess.run([path], capture_output=True, text=True, timeout=timeout, cwd=REF)
    return r.returncode, r.stdout + r.stderr


def test_unit_suite_reference_engine():
    rc, out = _run(_bin("unit_tests_ref"), 300)
    assert rc == 0, out[-3000:]
    assert "test cases: 85 | 85 passed | 0 failed" in out


def test_acceptance_reference_engine():
    rc, out = _run(_bin("acceptance_ref"), 600)
    assert rc == 0, out[-3000:]
    assert "all hard criteria passed" in out


@pytest.mark.gpu
def test_unit_suite_gpu_engine():
    """All 85 reference unit cases, engine.hpp served by the sm_100a kernels."""
    rc, out = _run(_bin("unit_tests_kk"), 600)
    assert rc == 0, out[-3000:]
    assert "test cases: 85 | 85 passed | 0 failed" in out


@pytest.mark.gpu
def test_acceptance_gpu_engine():
    """Acceptance criteria (oracle equivalence over 500 instances x every
    accumulator x scheme x worker count, determinism, L2 escalation,
    compression, reuse...) with engine.hpp served by the GPU."""
    rc, out = _run(_bin("acceptance_kk"), 900)
    print(out)
    assert rc == 0, out[-3000:]
    assert "all hard criteria passed" in out
