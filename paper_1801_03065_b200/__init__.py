"""kkSpGEMM on B200 — host-side mirror of the reference handle API.

The product is ``libkkspgemm.so`` (sm_100a kernels behind the C ABI declared in
``include/kkspgemm.h``).  This module binds that ABI with ctypes and mirrors
the reference's C++ interface (``proj/include/spgemm/engine.hpp:12-103``) with
the same names, argument meaning and error behaviour, so tests read like the
reference's own tests:

    SpgemmConfig, symbolic(a, b, cfg) -> SpgemmHandle,
    numeric(a, b, handle) -> CsrMatrix, multiply(a, b, cfg) -> MultiplyResult,
    resolve_config(...), flat_position(prefix, t)

and the reference's exceptions (``common.hpp:16-52``): ContractError,
ReuseError, PoolSizingError (all SpgemmError).  Device memory and streams come
from PyTorch (plumbing); every computation runs in the CUDA library.  There is
no CPU fallback: without a GPU, compute calls raise SpgemmError.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libkkspgemm.so")
GEN_PATH = os.path.join(_PKG, "libkkgen.so")

# ---- exceptions (common.hpp:16-52) -------------------------------------------


class SpgemmError(RuntimeError):
    pass


class ContractError(SpgemmError):
    pass


class ReuseError(SpgemmError):
    pass


class PoolSizingError(SpgemmError):
    pass


class InternalError(SpgemmError):  # std::logic_error in the reference
    pass


class CudaError(SpgemmError):
    pass


SPG_OK, SPG_ERR_CONTRACT, SPG_ERR_REUSE, SPG_ERR_POOL_SIZING = 0, 1, 2, 4
SPG_ERR_INTERNAL, SPG_ERR_CUDA, SPG_ERR_NOMEM = 5, 6, 7
_ERRORS = {
    SPG_ERR_CONTRACT: ContractError,
    SPG_ERR_REUSE: ReuseError,
    SPG_ERR_POOL_SIZING: PoolSizingError,
    SPG_ERR_INTERNAL: InternalError,
    SPG_ERR_CUDA: CudaError,
    SPG_ERR_NOMEM: CudaError,
}

# ---- enums (engine.hpp:14-33, compression.hpp:60, memory_pool.hpp:16) --------


class Scheme:
    ThreadSequential = 0
    ThreadFlatParallel = 1


class AccumulatorKind:
    Auto = 0
    LL = 1
    LP = 2
    Dense = 3


class CompressionMode:
    Auto = 0
    Always = 1
    Never = 2


class PoolMode:
    One2One = 0
    Many2Many = 1


class Phase:
    Symbolic = 0
    Numeric = 1


# ---- C structs (include/kkspgemm.h) -------------------------------------------


class _Csr(C.Structure):
    _fields_ = [("num_rows", C.c_int32), ("num_cols", C.c_int32), ("nnz", C.c_int64),
                ("row_offsets", C.c_void_p), ("col_indices", C.c_void_p), ("values", C.c_void_p)]


class _Config(C.Structure):
    _fields_ = [("scheme", C.c_int32), ("accumulator", C.c_int32), ("l1_capacity", C.c_int32),
                ("dense_cutoff_k", C.c_int32), ("avg_flops_cutoff", C.c_double),
                ("lp_max_occupancy", C.c_double), ("compression_gate", C.c_double),
                ("compression", C.c_int32), ("collapse_divisor", C.c_int32),
                ("worker_count", C.c_int32), ("sort_output", C.c_int32), ("row_block", C.c_int32),
                ("pool_mode", C.c_int32), ("pool_budget_bytes", C.c_int64)]


class _Resolved(C.Structure):
    _fields_ = [("accumulator", C.c_int32), ("scheme", C.c_int32), ("l1_capacity", C.c_int32),
                ("effective_k", C.c_int32), ("l2_capacity", C.c_int32)]


class _PhaseStats(C.Structure):
    _fields_ = [("ms", C.c_double), ("pool_allocations", C.c_int64), ("l2_inserts", C.c_int64)]


class _Flops(C.Structure):
    _fields_ = [("total_flops", C.c_int64), ("max_row_flops", C.c_int64),
                ("avg_degree_a", C.c_double), ("avg_row_flops", C.c_double)]


class _Report(C.Structure):
    _fields_ = [("cf", C.c_double), ("cmrf", C.c_double), ("compressed_flops", C.c_int64),
                ("compressed_max_row_flops", C.c_int64), ("applied", C.c_int32)]


class _Info(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("k", C.c_int32),
                ("nnz_a", C.c_int64), ("nnz_b", C.c_int64), ("nnz_c", C.c_int64),
                ("flops", _Flops), ("compression", _Report), ("max_row_size", C.c_int64),
                ("avg_row_size", C.c_double), ("avg_row_size_estimate", C.c_double),
                ("symbolic_choice", _Resolved), ("numeric_choice", _Resolved),
                ("config", _Config), ("symbolic_stats", _PhaseStats), ("compress_ms", C.c_double),
                ("d_c_row_offsets", C.c_void_p), ("d_per_row_flops", C.c_void_p),
                ("compressed_nnz_b", C.c_int64), ("heavy_path", C.c_int32), ("b_sorted", C.c_int32)]


class _Desc(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("k", C.c_int32),
                ("nnz_a", C.c_int64), ("nnz_b", C.c_int64), ("c_row_offsets", C.c_void_p),
                ("flops", _Flops), ("compression", _Report), ("max_row_size", C.c_int64),
                ("avg_row_size", C.c_double), ("avg_row_size_estimate", C.c_double),
                ("symbolic_choice", _Resolved), ("numeric_choice", _Resolved),
                ("config", _Config), ("symbolic_stats", _PhaseStats), ("compress_ms", C.c_double),
                ("per_row_flops", C.c_void_p)]


# every symbol include/kkspgemm.h declares (checked by tests/test_abi.py)
EXPORTED_SYMBOLS = (
    "spg_last_error", "spg_config_init", "spg_resolve_config", "spg_flat_position",
    "spg_symbolic", "spg_numeric", "spg_handle_info_get", "spg_handle_copy_row_offsets",
    "spg_handle_copy_per_row_flops", "spg_handle_copy_row_offsets_device", "spg_handle_set_numeric", "spg_handle_import",
    "spg_handle_check", "spg_handle_destroy", "spg_sort_rows", "spg_kernel_launch_count", "spg_row_digests",
    "spg_row_flops", "spg_handle_replay_state", "spg_numeric_rows", "spg_transpose",
)

_lib_handle = None


def lib() -> C.CDLL:
    """Load libkkspgemm.so.  Fails loudly when the extension was not built."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1801_03065_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.spg_last_error.restype = C.c_char_p
        L.spg_kernel_launch_count.restype = C.c_int64
        L.spg_handle_destroy.restype = None
        L.spg_handle_replay_state.restype = C.c_int
        L.spg_transpose.restype = C.c_int
        L.spg_transpose.argtypes = [C.POINTER(_Csr), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.spg_handle_replay_state.argtypes = [C.c_void_p]
        for name in ("spg_config_init", "spg_resolve_config", "spg_flat_position", "spg_symbolic",
                     "spg_numeric", "spg_handle_info_get", "spg_handle_copy_row_offsets",
                     "spg_handle_copy_per_row_flops", "spg_handle_copy_row_offsets_device", "spg_handle_set_numeric",
                     "spg_handle_import", "spg_handle_check", "spg_sort_rows", "spg_row_flops"):
            getattr(L, name).restype = C.c_int
        L.spg_symbolic.argtypes = [C.POINTER(_Csr), C.POINTER(_Csr), C.POINTER(_Config),
                                   C.POINTER(C.c_void_p), C.c_void_p]
        L.spg_numeric.argtypes = [C.c_void_p, C.POINTER(_Csr), C.POINTER(_Csr), C.c_void_p,
                                  C.c_void_p, C.POINTER(_PhaseStats), C.c_void_p]
        L.spg_numeric_rows.restype = C.c_int
        L.spg_numeric_rows.argtypes = [C.c_void_p, C.POINTER(_Csr), C.POINTER(_Csr), C.c_int32, C.c_int32,
                                       C.c_void_p, C.c_void_p, C.POINTER(_PhaseStats), C.c_void_p]
        L.spg_handle_info_get.argtypes = [C.c_void_p, C.POINTER(_Info)]
        L.spg_handle_copy_row_offsets.argtypes = [C.c_void_p, C.c_void_p]
        L.spg_handle_copy_per_row_flops.argtypes = [C.c_void_p, C.c_void_p]
        L.spg_handle_copy_row_offsets_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.spg_handle_set_numeric.argtypes = [C.c_void_p, C.POINTER(_Config), C.POINTER(_Resolved)]
        L.spg_handle_import.argtypes = [C.POINTER(_Desc), C.POINTER(C.c_void_p), C.c_void_p]
        L.spg_handle_check.argtypes = [C.c_void_p]
        L.spg_handle_destroy.argtypes = [C.c_void_p]
        L.spg_resolve_config.argtypes = [C.c_int32, C.c_int32, C.POINTER(_Flops), C.POINTER(_Report),
                                         C.POINTER(_Config), C.c_int64, C.POINTER(_Resolved)]
        L.spg_flat_position.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int64)]
        L.spg_sort_rows.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.spg_row_flops.argtypes = [C.POINTER(_Csr), C.POINTER(_Csr), C.c_void_p, C.c_void_p]
        L.spg_row_digests.restype = C.c_int
        L.spg_row_digests.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib_handle = L
    return _lib_handle


def _check(rc: int) -> None:
    if rc != SPG_OK:
        msg = lib().spg_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, SpgemmError)(msg)


def kernel_launch_count() -> int:
    return int(lib().spg_kernel_launch_count())


# ---- data model (csr_matrix.hpp:19-56) ------------------------------------------


@dataclasses.dataclass
class CsrMatrix:
    """Host CSR matrix: int64 row_offsets, int32 col_indices, fp64 values."""
    num_rows: int
    num_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    sorted_rows: bool = False

    def nnz(self) -> int:
        return int(self.row_offsets[-1] - self.row_offsets[0]) if len(self.row_offsets) else 0

    def row_size(self, i: int) -> int:
        return int(self.row_offsets[i + 1] - self.row_offsets[i])

    def to_device(self, device="cuda") -> "DeviceCsr":
        import torch
        return DeviceCsr(self.num_rows, self.num_cols,
                         torch.from_numpy(np.ascontiguousarray(self.row_offsets, np.int64)).to(device),
                         torch.from_numpy(np.ascontiguousarray(self.col_indices, np.int32)).to(device),
                         torch.from_numpy(np.ascontiguousarray(self.values, np.float64)).to(device),
                         self.sorted_rows)

    @staticmethod
    def from_scipy(s, sorted_rows: bool = True) -> "CsrMatrix":
        s = s.tocsr()
        return CsrMatrix(s.shape[0], s.shape[1], s.indptr.astype(np.int64), s.indices.astype(np.int32),
                         s.data.astype(np.float64), sorted_rows)


@dataclasses.dataclass
class DeviceCsr:
    """Device CSR view over torch CUDA tensors (or a row block of one)."""
    num_rows: int
    num_cols: int
    row_offsets: "object"  # torch.int64 [num_rows+1]
    col_indices: "object"  # torch.int32
    values: "object"       # torch.float64
    sorted_rows: bool = False
    nnz_: Optional[int] = None

    def nnz(self) -> int:
        if self.nnz_ is None:
            ro = self.row_offsets
            self.nnz_ = int(ro[-1].item() - ro[0].item()) if ro.numel() else 0
        return self.nnz_

    def row_block(self, lo: int, hi: int) -> "DeviceCsr":
        """Rows [lo, hi) as a view: row_offsets slice, shared col/val arrays."""
        return DeviceCsr(hi - lo, self.num_cols, self.row_offsets[lo:hi + 1], self.col_indices,
                         self.values, self.sorted_rows)

    def _c(self) -> _Csr:
        return _Csr(self.num_rows, self.num_cols, self.nnz(), self.row_offsets.data_ptr(),
                    self.col_indices.data_ptr() if self.col_indices.numel() else None,
                    self.values.data_ptr() if self.values is not None and self.values.numel() else None)

    def to_host(self) -> CsrMatrix:
        ro = self.row_offsets.cpu().numpy().astype(np.int64)
        base = int(ro[0]) if len(ro) else 0
        n = self.nnz()
        return CsrMatrix(self.num_rows, self.num_cols, ro - base,
                         self.col_indices[base:base + n].cpu().numpy(),
                         self.values[base:base + n].cpu().numpy(), self.sorted_rows)


# ---- config / handle (engine.hpp:18-72) ----------------------------------------


@dataclasses.dataclass
class SpgemmConfig:
    scheme: int = Scheme.ThreadSequential
    accumulator: int = AccumulatorKind.Auto
    l1_capacity: int = 0
    dense_cutoff_k: int = 250_000
    avg_flops_cutoff: float = 256.0
    lp_max_occupancy: float = 0.5
    compression_gate: float = 0.15
    compression: int = CompressionMode.Auto
    collapse_divisor: int = 8
    worker_count: int = 1
    sort_output: bool = False
    row_block: int = 512
    pool_mode: int = PoolMode.One2One
    pool_budget_bytes: int = 1 << 30

    def _c(self) -> _Config:
        return _Config(self.scheme, self.accumulator, self.l1_capacity, self.dense_cutoff_k,
                       self.avg_flops_cutoff, self.lp_max_occupancy, self.compression_gate,
                       self.compression, self.collapse_divisor, self.worker_count,
                       int(bool(self.sort_output)), self.row_block, self.pool_mode,
                       self.pool_budget_bytes)

    @staticmethod
    def _from_c(c: _Config) -> "SpgemmConfig":
        return SpgemmConfig(c.scheme, c.accumulator, c.l1_capacity, c.dense_cutoff_k,
                            c.avg_flops_cutoff, c.lp_max_occupancy, c.compression_gate,
                            c.compression, c.collapse_divisor, c.worker_count, bool(c.sort_output),
                            c.row_block, c.pool_mode, c.pool_budget_bytes)


@dataclasses.dataclass
class ResolvedConfig:
    accumulator: int
    scheme: int
    l1_capacity: int
    effective_k: int
    l2_capacity: int

    @staticmethod
    def _from_c(r: _Resolved) -> "ResolvedConfig":
        return ResolvedConfig(r.accumulator, r.scheme, r.l1_capacity, r.effective_k, r.l2_capacity)

    def _c(self) -> _Resolved:
        return _Resolved(self.accumulator, self.scheme, self.l1_capacity, self.effective_k,
                         self.l2_capacity)


@dataclasses.dataclass
class PhaseStats:
    ms: float = 0.0
    pool_allocations: int = 0
    l2_inserts: int = 0


@dataclasses.dataclass
class FlopsStats:
    total_flops: int = 0
    max_row_flops: int = 0
    avg_degree_a: float = 0.0
    avg_row_flops: float = 0.0
    per_row_flops: Optional[np.ndarray] = None


@dataclasses.dataclass
class CompressionReport:
    cf: float = 1.0
    cmrf: float = 1.0
    compressed_flops: int = 0
    compressed_max_row_flops: int = 0
    applied: bool = False


class SpgemmHandle:
    """Owns the device structure of C (row offsets) plus every host field of
    the reference SpgemmHandle (engine.hpp:53-72)."""

    def __init__(self, ptr: int):
        self._ptr = C.c_void_p(ptr)

    def __del__(self):
        try:
            if self._ptr and self._ptr.value:
                lib().spg_handle_destroy(self._ptr)
                self._ptr = C.c_void_p(None)
        except Exception:
            pass

    def _info(self) -> _Info:
        info = _Info()
        _check(lib().spg_handle_info_get(self._ptr, C.byref(info)))
        return info

    @property
    def m(self): return self._info().m
    @property
    def n(self): return self._info().n
    @property
    def k(self): return self._info().k
    @property
    def nnz_a(self): return self._info().nnz_a
    @property
    def nnz_b(self): return self._info().nnz_b

    def nnz_c(self) -> int:
        return int(self._info().nnz_c)

    @property
    def max_row_size(self): return int(self._info().max_row_size)

    @property
    def replay_state(self) -> int:
        """0 hashing only, 1 replay eligible, 2 slot map recorded (kk_replay.cu)."""
        return int(lib().spg_handle_replay_state(self._ptr))
    @property
    def heavy_path(self) -> int:
        """Rows beyond the warp tables: 0 none, 1 hashed buckets, 2 column slabs."""
        return int(self._info().heavy_path)

    @property
    def avg_row_size(self): return float(self._info().avg_row_size)
    @property
    def avg_row_size_estimate(self): return float(self._info().avg_row_size_estimate)
    @property
    def compress_ms(self): return float(self._info().compress_ms)

    @property
    def flops(self) -> FlopsStats:
        f = self._info().flops
        return FlopsStats(f.total_flops, f.max_row_flops, f.avg_degree_a, f.avg_row_flops)

    def per_row_flops(self) -> np.ndarray:
        out = np.empty(self.m, dtype=np.int64)
        _check(lib().spg_handle_copy_per_row_flops(self._ptr, out.ctypes.data))
        return out

    @property
    def compression(self) -> CompressionReport:
        r = self._info().compression
        return CompressionReport(r.cf, r.cmrf, r.compressed_flops, r.compressed_max_row_flops,
                                 bool(r.applied))

    @property
    def symbolic_choice(self) -> ResolvedConfig:
        return ResolvedConfig._from_c(self._info().symbolic_choice)

    @property
    def numeric_choice(self) -> ResolvedConfig:
        return ResolvedConfig._from_c(self._info().numeric_choice)

    @property
    def config(self) -> SpgemmConfig:
        return SpgemmConfig._from_c(self._info().config)

    @property
    def symbolic_stats(self) -> PhaseStats:
        s = self._info().symbolic_stats
        return PhaseStats(s.ms, s.pool_allocations, s.l2_inserts)

    @property
    def c_row_offsets(self) -> np.ndarray:
        out = np.empty(self.m + 1, dtype=np.int64)
        _check(lib().spg_handle_copy_row_offsets(self._ptr, out.ctypes.data))
        return out

    def device_row_offsets(self, stream=None):
        """The handle's row offsets as a new torch CUDA tensor (device copy)."""
        import torch
        t = torch.empty(self.m + 1, dtype=torch.int64, device="cuda")
        _check(lib().spg_handle_copy_row_offsets_device(self._ptr, t.data_ptr(), _stream_ptr(stream)))
        return t

    def set_numeric(self, config: Optional[SpgemmConfig] = None,
                    numeric_choice: Optional[ResolvedConfig] = None) -> None:
        """Edit handle.config / handle.numeric_choice (acceptance_main.cpp:417-425)."""
        _check(lib().spg_handle_set_numeric(self._ptr, C.byref(config._c()) if config else None,
                                            C.byref(numeric_choice._c()) if numeric_choice else None))

    def check(self) -> None:
        _check(lib().spg_handle_check(self._ptr))


@dataclasses.dataclass
class MultiplyResult:
    c: DeviceCsr
    handle: SpgemmHandle
    numeric_stats: PhaseStats


def _dev(x, device="cuda") -> DeviceCsr:
    if isinstance(x, DeviceCsr):
        return x
    if isinstance(x, CsrMatrix):
        return x.to_device(device)
    raise TypeError(f"expected CsrMatrix or DeviceCsr, got {type(x)}")


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


# ---- the handle API (engine.hpp:86-103) -------------------------------------------


def resolve_config(phase: int, k: int, stats: FlopsStats, report: CompressionReport,
                   cfg: SpgemmConfig, row_upper_bound: int) -> ResolvedConfig:
    out = _Resolved()
    f = _Flops(stats.total_flops, stats.max_row_flops, stats.avg_degree_a, stats.avg_row_flops)
    r = _Report(report.cf, report.cmrf, report.compressed_flops, report.compressed_max_row_flops,
                int(report.applied))
    _check(lib().spg_resolve_config(phase, k, C.byref(f), C.byref(r), C.byref(cfg._c()),
                                    row_upper_bound, C.byref(out)))
    return ResolvedConfig._from_c(out)


def flat_position(prefix, t: int):
    p = np.ascontiguousarray(prefix, dtype=np.int64)
    seg, off = C.c_int32(), C.c_int64()
    _check(lib().spg_flat_position(p.ctypes.data, len(p), t, C.byref(seg), C.byref(off)))
    return int(seg.value), int(off.value)


def symbolic(a, b, cfg: Optional[SpgemmConfig] = None, stream=None) -> SpgemmHandle:
    if a.num_cols != b.num_rows:  # checked again by the library
        raise ContractError("symbolic: inner dimensions do not match")
    da, db = _dev(a), _dev(b)
    ptr = C.c_void_p()
    cfgc = (cfg or SpgemmConfig())._c()
    _check(lib().spg_symbolic(C.byref(da._c()), C.byref(db._c()), C.byref(cfgc), C.byref(ptr),
                              _stream_ptr(stream)))
    return SpgemmHandle(ptr.value)


def numeric(a, b, handle: SpgemmHandle, stats: Optional[PhaseStats] = None, stream=None,
            out=None) -> DeviceCsr:
    """Fill C = A*B in the handle's structure.  Returns C as a DeviceCsr
    (row offsets copied from the handle).  `out` = (cols, vals) tensors to
    reuse; `stats` (a PhaseStats) makes the call synchronous and fills it."""
    import torch
    info = handle._info()
    if a.num_rows != info.m or a.num_cols != info.n or b.num_rows != info.n or b.num_cols != info.k:
        raise ReuseError("numeric: operands do not match the symbolic handle")
    da, db = _dev(a), _dev(b)
    nnz = int(info.nnz_c)
    if out is None:
        cols = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
        vals = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
    else:
        cols, vals = out
    st = _PhaseStats()
    _check(lib().spg_numeric(handle._ptr, C.byref(da._c()), C.byref(db._c()), cols.data_ptr(),
                             vals.data_ptr(), C.byref(st) if stats is not None else None,
                             _stream_ptr(stream)))
    if stats is not None:
        stats.ms, stats.pool_allocations, stats.l2_inserts = st.ms, st.pool_allocations, st.l2_inserts
    rowptr = handle.device_row_offsets(stream)
    return DeviceCsr(info.m, info.k, rowptr, cols[:nnz] if nnz else cols[:0],
                     vals[:nnz] if nnz else vals[:0], bool(info.config.sort_output), nnz)


def numeric_rows(a, b, handle: SpgemmHandle, row_begin: int, row_end: int, cols, vals,
                 stats: Optional[PhaseStats] = None, stream=None) -> None:
    """numeric restricted to C rows [row_begin, row_end), into the full C
    buffers `cols`/`vals` (nnz_c entries each; other rows untouched)."""
    info = handle._info()
    if a.num_rows != info.m or a.num_cols != info.n or b.num_rows != info.n or b.num_cols != info.k:
        raise ReuseError("numeric: operands do not match the symbolic handle")
    da, db = _dev(a), _dev(b)
    st = _PhaseStats()
    _check(lib().spg_numeric_rows(handle._ptr, C.byref(da._c()), C.byref(db._c()), row_begin, row_end,
                                  cols.data_ptr(), vals.data_ptr(), C.byref(st) if stats is not None else None,
                                  _stream_ptr(stream)))
    if stats is not None:
        stats.ms, stats.pool_allocations, stats.l2_inserts = st.ms, st.pool_allocations, st.l2_inserts


def multiply(a, b, cfg: Optional[SpgemmConfig] = None, stream=None) -> MultiplyResult:
    h = symbolic(a, b, cfg, stream)
    st = PhaseStats()
    c = numeric(a, b, h, st, stream)
    return MultiplyResult(c, h, st)


def import_handle(m: int, n: int, k: int, nnz_a: int, nnz_b: int, c_row_offsets: np.ndarray,
                  numeric_choice: ResolvedConfig, config: SpgemmConfig, **fields) -> SpgemmHandle:
    """Rebuild a device handle from host fields (the engine.hpp shim path)."""
    ro = np.ascontiguousarray(c_row_offsets, dtype=np.int64)
    d = _Desc()
    d.m, d.n, d.k, d.nnz_a, d.nnz_b = m, n, k, nnz_a, nnz_b
    d.c_row_offsets = ro.ctypes.data
    d.max_row_size = int(np.max(np.diff(ro))) if m > 0 else 0
    d.numeric_choice = numeric_choice._c()
    d.config = config._c()
    ptr = C.c_void_p()
    _check(lib().spg_handle_import(C.byref(d), C.byref(ptr), _stream_ptr(None)))
    return SpgemmHandle(ptr.value)


def row_flops(a, b, stream=None):
    """Per-row multiplication counts on the device (torch.int64 [m])."""
    import torch
    da, db = _dev(a), _dev(b)
    out = torch.empty(max(da.num_rows, 1), dtype=torch.int64, device=da.row_offsets.device)
    _check(lib().spg_row_flops(C.byref(da._c()), C.byref(db._c()), out.data_ptr(), _stream_ptr(stream)))
    return out[:da.num_rows]


def transpose(a, stream=None) -> DeviceCsr:
    """A^T on the device (csr_matrix.cpp:82-108 order), e.g. R = P^T."""
    import torch
    da = _dev(a)
    dev = da.row_offsets.device
    nnz = da.nnz()
    ro = torch.empty(da.num_cols + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    v = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    _check(lib().spg_transpose(C.byref(da._c()), ro.data_ptr(), ci.data_ptr(), v.data_ptr(), _stream_ptr(stream)))
    return DeviceCsr(da.num_cols, da.num_rows, ro, ci[:nnz], v[:nnz], True, nnz)


def row_digests(c: DeviceCsr, stream=None):
    """Per-row canonical digests of a device CSR (torch.int64 [m] holding the
    uint64 bits): order-independent hash of each row's (column, value bits)
    set and length — the device side of canonicalize + compare_canonical
    (oracle.cpp:105-159); the oracle computes the same function."""
    import torch
    out = torch.empty(max(c.num_rows, 1), dtype=torch.int64, device=c.row_offsets.device)
    _check(lib().spg_row_digests(c.num_rows, c.row_offsets.data_ptr(), c.col_indices.data_ptr(),
                                 c.values.data_ptr(), out.data_ptr(), _stream_ptr(stream)))
    return out[:c.num_rows]


def sort_rows(c: DeviceCsr, stream=None) -> DeviceCsr:
    _check(lib().spg_sort_rows(c.num_rows, c.row_offsets.data_ptr(), c.col_indices.data_ptr(),
                               c.values.data_ptr(), _stream_ptr(stream)))
    c.sorted_rows = True
    return c


from . import generators  # noqa: E402,F401
