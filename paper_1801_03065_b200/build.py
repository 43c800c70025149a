"""Build the in-tree native libraries.

* ``libkkspgemm.so`` — the product: sm_100a kernels + C ABI (include/kkspgemm.h),
  compiled with ``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo``.
* ``libkkgen.so`` — host-side input generators (bench/test plumbing, shared by
  the GPU path and the oracle so both see byte-identical inputs).
* ``oracle/`` — the parity checkers (``make -C oracle``); the reference build
  (``oracle/_ref``) only when /root/reference is present.

Everything is written in-tree so the built ``.so`` files travel to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libkkspgemm.so")
GEN = os.path.join(PKG, "libkkgen.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_kkspgemm(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, f) for f in ("kk_api.cu", "kk_kernels.cu", "kk_fast.cu", "kk_heavy.cu", "kk_slab.cu", "kk_replay.cu", "kk_tiny.cu")]
    deps = srcs + [os.path.join(CSRC, f) for f in ("kk_device.cuh", "kk_internal.h")] + [
        os.path.join(ROOT, "include", "kkspgemm.h")]
    if force or _stale(LIB, deps):
        extra = os.environ.get("KK_NVCC_DEFS", "").split()  # e.g. -DKK_SLAB_PROF (profiling builds)
        cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), *srcs, "-o", LIB]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
    return LIB


def build_generators(force: bool = False) -> str:
    src = os.path.join(CSRC, "generators.cpp")
    if force or _stale(GEN, [src]):
        subprocess.run(["g++", "-std=c++20", "-O3", "-fPIC", "-shared", src, "-o", GEN], check=True)
    return GEN


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        # the reference library, its own test suites against it, and the same
        # suites against libkkspgemm.so through the engine.hpp shim
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref", "reftests", "kktests"],
                       check=True)


def build_all(force: bool = False) -> None:
    build_kkspgemm(force)
    build_generators(force)
    build_oracle()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
