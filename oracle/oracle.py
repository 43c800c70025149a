"""TEST INFRASTRUCTURE ONLY — Python bindings of the parity checkers.

* ``Oracle``   — oracle/liboracle.so, the C restatement (spgemm_oracle.c).
* ``Reference``— oracle/_ref/libspgemm_ref.so, the UNMODIFIED reference library
                 compiled from /root/reference/proj/src (present when it was
                 built in this container; the built .so travels to the GPU box).

Only tests/ (incl. tests/tools/), __graft_entry__.smoke() and the CPU-baseline
legs of bench.py (cpu_baseline, ``--impl reference``) and of its companion for
the other BASELINE configs, scripts/bench_configs.py, may import this module,
and only as the checker or the timed reference.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspgemm_ref.so")

_P = C.c_void_p


def _ptr(a):
    return a.ctypes.data if a is not None and a.size else None


class Oracle:
    """The C restatement of the reference hot path."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
        L = C.CDLL(ORACLE_SO)
        L.orc_max_rel_error.restype = C.c_double
        L.orc_max_rel_error.argtypes = [C.c_int64, _P, _P]
        for f, args in {
            "orc_flops_stats": [C.c_int32, _P, _P, _P, _P, _P, _P],
            "orc_compressed_row_sizes": [C.c_int32, C.c_int32, _P, _P, _P],
            "orc_decide_compression": [C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P, C.c_int64,
                                       C.c_double, C.c_int, _P, _P, _P],
            "orc_symbolic_row_sizes": [C.c_int32, C.c_int32, _P, _P, _P, _P, _P],
            "orc_numeric": [C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P],
            "orc_sort_rows": [C.c_int32, _P, _P, _P],
            "orc_resolve_config": [C.c_int, C.c_int32, C.c_double, C.c_int, C.c_int, C.c_int,
                                   C.c_int32, C.c_int32, C.c_double, C.c_int64, _P],
            "orc_row_digests": [C.c_int32, _P, _P, _P, _P],
            "orc_product_row_digests": [C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P, C.c_int, _P, _P],
        }.items():
            getattr(L, f).restype = C.c_int
            getattr(L, f).argtypes = args
        self.L = L

    @staticmethod
    def _norm(m):
        ro = np.ascontiguousarray(m.row_offsets, np.int64)
        return ro, np.ascontiguousarray(m.col_indices, np.int32), np.ascontiguousarray(m.values, np.float64)

    def flops_stats(self, a, b):
        ar, ac, _ = self._norm(a)
        br, _, _ = self._norm(b)
        per = np.empty(max(a.num_rows, 1), np.int64)
        tot, mx = C.c_int64(), C.c_int64()
        self.L.orc_flops_stats(a.num_rows, _ptr(ar), _ptr(ac), _ptr(br), _ptr(per), C.byref(tot), C.byref(mx))
        return per[:a.num_rows], tot.value, mx.value

    def compressed_row_sizes(self, b):
        br, bc, _ = self._norm(b)
        out = np.empty(max(b.num_rows, 1), np.int32)
        self.L.orc_compressed_row_sizes(b.num_rows, b.num_cols, _ptr(br), _ptr(bc), _ptr(out))
        return out[:b.num_rows]

    def decide_compression(self, a, b, gate=0.15, mode=0):
        ar, ac, _ = self._norm(a)
        br, bc, _ = self._norm(b)
        _, total, mxf = self.flops_stats(a, b)
        cf, cm, ap = C.c_int64(), C.c_int64(), C.c_int()
        self.L.orc_decide_compression(a.num_rows, b.num_rows, b.num_cols, _ptr(ar), _ptr(ac), _ptr(br),
                                      _ptr(bc), total, gate, mode, C.byref(cf), C.byref(cm), C.byref(ap))
        return {"compressed_flops": cf.value, "compressed_max_row_flops": cm.value,
                "applied": bool(ap.value),
                "cf": cf.value / total if total > 0 else 1.0,
                "cmrf": cm.value / mxf if mxf > 0 else 1.0}

    def symbolic_row_offsets(self, a, b):
        ar, ac, _ = self._norm(a)
        br, bc, _ = self._norm(b)
        sizes = np.empty(max(a.num_rows, 1), np.int64)
        self.L.orc_symbolic_row_sizes(a.num_rows, b.num_cols, _ptr(ar), _ptr(ac), _ptr(br), _ptr(bc), _ptr(sizes))
        ro = np.zeros(a.num_rows + 1, np.int64)
        np.cumsum(sizes[:a.num_rows], out=ro[1:])
        return ro

    def numeric(self, a, b, c_rowptr):
        """Raw (first-touch order) C cols/vals, bitwise the reference's output."""
        ar, ac, av = self._norm(a)
        br, bc, bv = self._norm(b)
        cr = np.ascontiguousarray(c_rowptr, np.int64)
        nnz = int(cr[-1] - cr[0])
        cols = np.empty(max(nnz, 1), np.int32)
        vals = np.empty(max(nnz, 1), np.float64)
        rc = self.L.orc_numeric(a.num_rows, b.num_cols, _ptr(ar), _ptr(ac), _ptr(av), _ptr(br), _ptr(bc),
                                _ptr(bv), _ptr(cr), _ptr(cols), _ptr(vals))
        if rc != 0:
            raise RuntimeError(f"orc_numeric failed ({rc})")
        return cols[:nnz], vals[:nnz]

    def multiply(self, a, b):
        ro = self.symbolic_row_offsets(a, b)
        cols, vals = self.numeric(a, b, ro)
        return ro, cols, vals

    def sort_rows(self, rowptr, cols, vals):
        cols = np.array(cols, np.int32, copy=True)
        vals = np.array(vals, np.float64, copy=True)
        ro = np.ascontiguousarray(rowptr, np.int64) - int(rowptr[0])
        self.L.orc_sort_rows(len(ro) - 1, _ptr(ro), _ptr(cols), _ptr(vals))
        return cols, vals

    def row_digests(self, m):
        """Per-row canonical digests of a CSR (order-independent; see spgemm_oracle.h)."""
        ro, ci, v = self._norm(m)
        out = np.empty(max(m.num_rows, 1), np.uint64)
        self.L.orc_row_digests(m.num_rows, _ptr(ro), _ptr(ci), _ptr(v), _ptr(out))
        return out[:m.num_rows]

    def product_row_digests(self, a, b, threads=None):
        """(digests, row sizes) of every row of C = A*B, formed by the numeric
        restatement in `threads` threads without storing C."""
        ar, ac, av = self._norm(a)
        br, bc, bv = self._norm(b)
        out = np.empty(max(a.num_rows, 1), np.uint64)
        sizes = np.empty(max(a.num_rows, 1), np.int64)
        rc = self.L.orc_product_row_digests(a.num_rows, b.num_cols, _ptr(ar), _ptr(ac), _ptr(av), _ptr(br),
                                            _ptr(bc), _ptr(bv), int(threads or os.cpu_count() or 1), _ptr(out),
                                            _ptr(sizes))
        assert rc == 0
        return out[:a.num_rows], sizes[:a.num_rows]

    def max_rel_error(self, expected, actual):
        e = np.ascontiguousarray(expected, np.float64)
        a = np.ascontiguousarray(actual, np.float64)
        assert e.shape == a.shape
        return self.L.orc_max_rel_error(len(e), _ptr(e), _ptr(a))

    def resolve_config(self, phase, k, avg_row_flops, applied, acc=0, scheme=0, l1=0,
                       dense_cutoff_k=250000, avg_flops_cutoff=256.0, bound=1):
        out = (C.c_int32 * 5)()
        self.L.orc_resolve_config(phase, k, avg_row_flops, int(applied), acc, scheme, l1, dense_cutoff_k,
                                  avg_flops_cutoff, bound, C.cast(out, _P))
        return dict(zip(("accumulator", "scheme", "l1_capacity", "effective_k", "l2_capacity"), list(out)))


# ---------------------------------------------------------------------------
class _RefCfg(C.Structure):
    _fields_ = [("scheme", C.c_int), ("accumulator", C.c_int), ("l1_capacity", C.c_int32),
                ("dense_cutoff_k", C.c_int32), ("avg_flops_cutoff", C.c_double),
                ("lp_max_occupancy", C.c_double), ("compression_gate", C.c_double),
                ("compression", C.c_int), ("collapse_divisor", C.c_int), ("worker_count", C.c_int),
                ("sort_output", C.c_int), ("row_block", C.c_int32), ("pool_mode", C.c_int),
                ("pool_budget_bytes", C.c_int64)]


class _RefInfo(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("k", C.c_int32), ("nnz_a", C.c_int64),
                ("nnz_b", C.c_int64), ("nnz_c", C.c_int64), ("total_flops", C.c_int64),
                ("max_row_flops", C.c_int64), ("avg_degree_a", C.c_double), ("avg_row_flops", C.c_double),
                ("cf", C.c_double), ("cmrf", C.c_double), ("compressed_flops", C.c_int64),
                ("compressed_max_row_flops", C.c_int64), ("applied", C.c_int32),
                ("max_row_size", C.c_int64), ("avg_row_size", C.c_double),
                ("avg_row_size_estimate", C.c_double),
                ("sym_acc", C.c_int32), ("sym_scheme", C.c_int32), ("sym_l1", C.c_int32),
                ("sym_effk", C.c_int32), ("sym_l2", C.c_int32),
                ("num_acc", C.c_int32), ("num_scheme", C.c_int32), ("num_l1", C.c_int32),
                ("num_effk", C.c_int32), ("num_l2", C.c_int32),
                ("sym_ms", C.c_double), ("sym_pool_allocations", C.c_int64), ("sym_l2_inserts", C.c_int64),
                ("compress_ms", C.c_double)]


class _RefStats(C.Structure):
    _fields_ = [("ms", C.c_double), ("pool_allocations", C.c_int64), ("l2_inserts", C.c_int64)]


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The unmodified reference library (oracle/_ref), wrapped by ref_capi.cpp."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            if os.path.isdir("/root/reference/proj/src"):
                subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)
            else:
                raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference)")
        L = C.CDLL(REF_SO)
        for f in ("ref_mat_new", "ref_build_csr", "ref_transpose", "ref_generate_synthetic", "ref_rng_new",
                  "ref_random_csr", "ref_shuffle_rows", "ref_synthetic_by_index", "ref_symbolic", "ref_read_mm"):
            getattr(L, f).restype = _P
        L.ref_mat_new.argtypes = [C.c_int32, C.c_int32, _P, _P, _P, C.c_int]
        L.ref_mat_free.argtypes = [_P]
        L.ref_mat_shape.argtypes = [_P, _P, _P, _P]
        L.ref_mat_export.argtypes = [_P, _P, _P, _P]
        L.ref_build_csr.argtypes = [C.c_int32, C.c_int32, C.c_int64, _P, _P, _P]
        L.ref_transpose.argtypes = [_P]
        L.ref_read_mm.argtypes = [C.c_char_p]
        L.ref_generate_synthetic.argtypes = [C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_uint64]
        L.ref_rng_new.argtypes = [C.c_uint64]
        L.ref_rng_free.argtypes = [_P]
        L.ref_rng_next.restype = C.c_uint64
        L.ref_rng_next.argtypes = [_P]
        L.ref_random_csr.argtypes = [_P, C.c_int32, C.c_int32, C.c_double]
        L.ref_shuffle_rows.argtypes = [_P, C.c_uint64]
        L.ref_synthetic_by_index.argtypes = [C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_uint64]
        L.ref_flops_stats.argtypes = [_P, _P, _P, _P, _P]
        L.ref_compressed_row_sizes.argtypes = [_P, _P]
        L.ref_decide_compression.argtypes = [_P, _P, C.c_double, C.c_int, _P, _P, _P, _P, _P]
        L.ref_cfg_default.argtypes = [_P]
        L.ref_cfg_default.restype = None
        L.ref_symbolic.argtypes = [_P, _P, _P]
        L.ref_handle_free.argtypes = [_P]
        L.ref_handle_info.argtypes = [_P, _P]
        L.ref_handle_rowptr.argtypes = [_P, _P]
        L.ref_handle_per_row_flops.argtypes = [_P, _P]
        L.ref_handle_set_workers.argtypes = [_P, C.c_int]
        L.ref_numeric.argtypes = [_P, _P, _P, _P, _P, _P]
        L.ref_multiply_ms.restype = C.c_double
        L.ref_multiply_ms.argtypes = [_P, _P, _P, _P]
        L.ref_gustavson_mults.restype = C.c_int64
        L.ref_gustavson_mults.argtypes = [_P, _P]
        L.ref_last_error.restype = C.c_char_p
        self.L = L

    # ---- matrices ----
    def mat(self, m):
        ro = np.ascontiguousarray(m.row_offsets, np.int64)
        ci = np.ascontiguousarray(m.col_indices, np.int32)
        v = np.ascontiguousarray(m.values, np.float64)
        return RefMat(self, self.L.ref_mat_new(m.num_rows, m.num_cols, _ptr(ro), _ptr(ci), _ptr(v),
                                               int(bool(m.sorted_rows))))

    def read_mm(self, path: str):
        """The reference's read_matrix_market (matrix_market.cpp:48-132)."""
        ptr = self.L.ref_read_mm(str(path).encode())
        if not ptr:
            raise ValueError(self.L.ref_last_error().decode())
        try:
            return self.export(ptr)
        finally:
            self.L.ref_mat_free(ptr)

    def export(self, handle):
        from paper_1801_03065_b200 import CsrMatrix
        r, c, n = C.c_int32(), C.c_int32(), C.c_int64()
        self.L.ref_mat_shape(handle, C.byref(r), C.byref(c), C.byref(n))
        ro = np.empty(r.value + 1, np.int64)
        ci = np.empty(max(n.value, 1), np.int32)
        v = np.empty(max(n.value, 1), np.float64)
        self.L.ref_mat_export(handle, _ptr(ro), _ptr(ci), _ptr(v))
        return CsrMatrix(r.value, c.value, ro, ci[:n.value], v[:n.value], False)

    def _own(self, ptr):
        if not ptr:
            raise RuntimeError(self.L.ref_last_error().decode())
        out = self.export(ptr)
        self.L.ref_mat_free(ptr)
        return out

    def generate_synthetic(self, kind, rows, cols, target, seed):
        m = self._own(self.L.ref_generate_synthetic(kind, rows, cols, target, seed))
        m.sorted_rows = True
        return m

    def build_csr(self, rows, cols, trips):
        r = np.array([t[0] for t in trips], np.int32)
        c = np.array([t[1] for t in trips], np.int32)
        v = np.array([t[2] for t in trips], np.float64)
        m = self._own(self.L.ref_build_csr(rows, cols, len(trips), _ptr(r), _ptr(c), _ptr(v)))
        m.sorted_rows = True
        return m

    def rng(self, seed):
        return RefRng(self, seed)

    def random_csr(self, rng, rows, cols, density):
        m = self._own(self.L.ref_random_csr(rng.ptr, rows, cols, density))
        m.sorted_rows = True
        return m

    def shuffle_rows(self, m, seed):
        rm = self.mat(m)
        out = self._own(self.L.ref_shuffle_rows(rm.ptr, seed))
        out.sorted_rows = False
        return out

    def synthetic_by_index(self, idx, rows, cols, target, seed):
        m = self._own(self.L.ref_synthetic_by_index(idx, rows, cols, target, seed))
        m.sorted_rows = True
        return m

    def cfg(self, **kw):
        c = _RefCfg()
        self.L.ref_cfg_default(C.byref(c))
        for k, v in kw.items():
            setattr(c, k, int(v) if isinstance(v, bool) else v)
        return c

    # ---- hot path ----
    def flops_stats(self, a, b):
        ra, rb = self.mat(a), self.mat(b)
        per = np.empty(max(a.num_rows, 1), np.int64)
        t, mx = C.c_int64(), C.c_int64()
        self.L.ref_flops_stats(ra.ptr, rb.ptr, _ptr(per), C.byref(t), C.byref(mx))
        return per[:a.num_rows], t.value, mx.value

    def compressed_row_sizes(self, b):
        rb = self.mat(b)
        out = np.empty(max(b.num_rows, 1), np.int32)
        self.L.ref_compressed_row_sizes(rb.ptr, _ptr(out))
        return out[:b.num_rows]

    def symbolic(self, a, b, **cfg):
        ra, rb = self.mat(a), self.mat(b)
        c = self.cfg(**cfg)
        h = self.L.ref_symbolic(ra.ptr, rb.ptr, C.byref(c))
        if not h:
            raise RuntimeError(self.L.ref_last_error().decode())
        return RefHandle(self, h, ra, rb)

    def multiply_ms(self, a, b, **cfg):
        ra, rb = self.mat(a), self.mat(b)
        c = self.cfg(**cfg)
        nnz = C.c_int64()
        ms = self.L.ref_multiply_ms(ra.ptr, rb.ptr, C.byref(c), C.byref(nnz))
        return ms, nnz.value


class RefMat:
    def __init__(self, ref, ptr):
        self.ref, self.ptr = ref, ptr

    def __del__(self):
        try:
            self.ref.L.ref_mat_free(self.ptr)
        except Exception:
            pass


class RefRng:
    def __init__(self, ref, seed):
        self.ref, self.ptr = ref, ref.L.ref_rng_new(seed)

    def next(self):
        return self.ref.L.ref_rng_next(self.ptr)

    def __del__(self):
        try:
            self.ref.L.ref_rng_free(self.ptr)
        except Exception:
            pass


class RefHandle:
    def __init__(self, ref, ptr, ra, rb):
        self.ref, self.ptr, self.ra, self.rb = ref, ptr, ra, rb

    def __del__(self):
        try:
            self.ref.L.ref_handle_free(self.ptr)
        except Exception:
            pass

    def info(self):
        i = _RefInfo()
        self.ref.L.ref_handle_info(self.ptr, C.byref(i))
        return {f: getattr(i, f) for f, _ in _RefInfo._fields_}

    def row_offsets(self):
        m = self.info()["m"]
        out = np.empty(m + 1, np.int64)
        self.ref.L.ref_handle_rowptr(self.ptr, _ptr(out))
        return out

    def per_row_flops(self):
        m = self.info()["m"]
        out = np.empty(max(m, 1), np.int64)
        self.ref.L.ref_handle_per_row_flops(self.ptr, _ptr(out))
        return out[:m]

    def set_workers(self, w):
        self.ref.L.ref_handle_set_workers(self.ptr, w)

    def numeric(self, a=None, b=None):
        """Raw C (first-touch order) from the reference numeric()."""
        ra = self.ref.mat(a) if a is not None else self.ra
        rb = self.ref.mat(b) if b is not None else self.rb
        nnz = self.info()["nnz_c"]
        cols = np.empty(max(nnz, 1), np.int32)
        vals = np.empty(max(nnz, 1), np.float64)
        st = _RefStats()
        rc = self.ref.L.ref_numeric(ra.ptr, rb.ptr, self.ptr, _ptr(cols), _ptr(vals), C.byref(st))
        if rc != 0:
            raise RuntimeError(f"ref numeric failed ({rc}): {self.ref.L.ref_last_error().decode()}")
        return cols[:nnz], vals[:nnz], {"ms": st.ms, "pool_allocations": st.pool_allocations,
                                        "l2_inserts": st.l2_inserts}


GEN_SO = os.path.join(HERE, "libgen.so")


def generators():
    """The BASELINE input generators built by the oracle Makefile from the same
    source as the product's (csrc/generators.cpp): bench.py's reference arm
    creates its inputs with these, so its process loads no product library."""
    if not os.path.exists(GEN_SO):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    from paper_1801_03065_b200.generators import Generators
    return Generators(GEN_SO)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"
