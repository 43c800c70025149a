"""Host-side generators for the BASELINE.json configurations (bench/test
plumbing).  Thin ctypes binding of csrc/generators.cpp; see that file for the
exact definitions."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import CsrMatrix, GEN_PATH

class Generators:
    """The generator functions over one build of csrc/generators.cpp: the
    package's libkkgen.so by default; bench.py's reference arm binds the copy
    the oracle Makefile builds (oracle/libgen.so), so that process loads no
    library of the product package."""

    def __init__(self, path: str = None):
        self.path = path or GEN_PATH
        self._L = None

    def _g(self):
        if self._L is None:
            if not os.path.exists(self.path):
                if self.path == GEN_PATH:
                    from .build import build_generators
                    build_generators()
                else:
                    raise FileNotFoundError(self.path)
            L = C.CDLL(self.path)
            for f in ("kkg_laplace2d", "kkg_laplace3d", "kkg_rmat", "kkg_aggregation", "kkg_transpose",
                      "kkg_read_mm"):
                getattr(L, f).restype = C.c_void_p
            L.kkg_read_mm.argtypes = [C.c_char_p, C.c_char_p, C.c_int32]
            L.kkg_laplace2d.argtypes = [C.c_int32, C.c_double, C.c_uint64]
            L.kkg_laplace3d.argtypes = [C.c_int32, C.c_double, C.c_uint64]
            L.kkg_rmat.argtypes = [C.c_int32, C.c_int32, C.c_uint64]
            L.kkg_aggregation.argtypes = [C.c_int32]
            L.kkg_transpose.argtypes = [C.c_void_p]
            L.kkg_shape.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
            L.kkg_export.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.kkg_free.argtypes = [C.c_void_p]
            self._L = L
        return self._L

    def take(self, ptr) -> CsrMatrix:
        L = self._g()
        r, c, n = C.c_int32(), C.c_int32(), C.c_int64()
        L.kkg_shape(ptr, C.byref(r), C.byref(c), C.byref(n))
        ro = np.empty(r.value + 1, np.int64)
        ci = np.empty(max(n.value, 1), np.int32)
        v = np.empty(max(n.value, 1), np.float64)
        L.kkg_export(ptr, ro.ctypes.data, ci.ctypes.data, v.ctypes.data)
        L.kkg_free(ptr)
        return CsrMatrix(r.value, c.value, ro, ci[:n.value], v[:n.value], True)

    def laplace2d(self, n: int, eps: float = 0.01, seed: int = 1801) -> CsrMatrix:
        """2D 5-point Laplacian on an n x n grid, weights {4,-1}*(1+eps*U(-1,1))."""
        return self.take(self._g().kkg_laplace2d(n, eps, seed))

    def laplace3d(self, n: int, eps: float = 0.01, seed: int = 1801) -> CsrMatrix:
        """3D 27-point Laplacian on an n^3 grid, weights {26,-1}*(1+eps*U(-1,1))."""
        return self.take(self._g().kkg_laplace3d(n, eps, seed))

    def rmat(self, scale: int, edge_factor: int = 16, seed: int = 1) -> CsrMatrix:
        """Graph500 R-MAT, duplicates summed, values U(-1,1)."""
        return self.take(self._g().kkg_rmat(scale, edge_factor, seed))

    def aggregation(self, n: int) -> CsrMatrix:
        """Piecewise-constant 2x2x2 aggregation prolongator for an n^3 grid."""
        return self.take(self._g().kkg_aggregation(n))

    @staticmethod
    def transpose(m: CsrMatrix) -> CsrMatrix:
        """R = P^T (csr_matrix.cpp:82-108 semantics: rows come out sorted)."""
        import scipy.sparse as sp
        s = sp.csr_matrix((m.values, m.col_indices, m.row_offsets - m.row_offsets[0]),
                          shape=(m.num_rows, m.num_cols))
        t = s.T.tocsr()
        t.sort_indices()
        return CsrMatrix(t.shape[0], t.shape[1], t.indptr.astype(np.int64), t.indices.astype(np.int32),
                         t.data.astype(np.float64), True)

    def read_matrix_market(self, path: str) -> CsrMatrix:
        """MatrixMarket coordinate file -> CsrMatrix (coordinate real/integer/
        pattern, general/symmetric, duplicates summed; csrc/generators.cpp
        read_mm).  Raises ValueError (the reference's ParseError/IoError)."""
        err = C.create_string_buffer(512)
        ptr = self._g().kkg_read_mm(os.fsencode(path), err, len(err))
        if not ptr:
            raise ValueError(err.value.decode())
        return self.take(ptr)

    def config_matrices(self, cfg: int, scale: float = 1.0):
        """Operands of BASELINE.json configs 1..5 (1-based, as SURVEY §8d lists
        them).  Returns a dict with A, B (and R, P for config 3)."""
        if cfg == 1:
            a = self.laplace2d(int(1000 * scale), 0.01, 1801)
            return {"A": a, "B": a}
        if cfg == 2:
            a = self.laplace3d(int(160 * scale), 0.01, 1801)
            return {"A": a, "B": a}
        if cfg == 3:
            n = int(128 * scale)
            a = self.laplace3d(n, 0.01, 1801)
            p = self.aggregation(n)
            return {"A": a, "P": p, "R": self.transpose(p)}
        if cfg == 4:
            a = self.rmat(int(round(20 + np.log2(scale))) if scale != 1.0 else 20, 16, 1)
            return {"A": a, "B": a}
        if cfg == 5:
            a = self.laplace3d(int(200 * scale), 0.01, 1801)
            return {"A": a, "B": a}
        raise ValueError(cfg)


_default = Generators()
laplace2d = _default.laplace2d
laplace3d = _default.laplace3d
rmat = _default.rmat
aggregation = _default.aggregation
transpose = Generators.transpose
read_matrix_market = _default.read_matrix_market
config_matrices = _default.config_matrices


def write_matrix_market(m: CsrMatrix, path: str) -> None:
    """General real coordinate file, 1-based, %.17g values (round-trips)."""
    base = int(m.row_offsets[0]) if len(m.row_offsets) else 0
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{m.num_rows} {m.num_cols} {m.nnz()}\n")
        for i in range(m.num_rows):
            for q in range(int(m.row_offsets[i]) - base, int(m.row_offsets[i + 1]) - base):
                f.write(f"{i + 1} {int(m.col_indices[q]) + 1} {float(m.values[q]):.17g}\n")
