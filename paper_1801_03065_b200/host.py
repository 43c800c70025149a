"""Host-memory multiply with copy/compute overlap (the reference's
`multiply(const CsrMatrix&, const CsrMatrix&, const SpgemmConfig&)`,
engine.hpp:100-103, for callers whose matrices live in host memory).

The reference is a CPU library: its multiply reads host CSR arrays and returns
a host CSR.  On a B200 the end-to-end cost of that call is dominated by the
host link (C is typically 4-5x larger than A), so the host path is organised
around the copies:

  * the operands' structure (row offsets, columns) is uploaded first and their
    values on a second stream, overlapping the symbolic phase (which reads
    structure only); for C = A*A the values go in row chunks and each block
    of C waits only for the chunks up to the last row it references;
  * a matrix passed as both A and B (C = A*A) is uploaded once; `a_rows`
    names A as a row block of B (the row-sharded multi-GPU case) so only B
    travels, and only B's row offsets plus the rows in the block's column band
    (a shard of a banded operator needs its slab and a halo);
  * one symbolic pass over all of A (C's size is then known and, unless the
    caller passes output buffers, the pinned output comes from torch's host
    caching allocator); the numeric pass then runs in row blocks
    (spg_numeric_rows) and block k's C is copied out on the copy stream while
    block k+1 computes.

Inputs must be in pinned host memory (PinnedCsr) for the copies to be
asynchronous.  Everything below the Python orchestration is the C ABI.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Tuple

import numpy as np

from . import CsrMatrix, DeviceCsr, SpgemmConfig, numeric_rows, symbolic

_copy_streams = {}


def _copy_stream(dev):
    import torch
    s = _copy_streams.get(dev.index)
    if s is None:
        s = torch.cuda.Stream(device=dev)
        _copy_streams[dev.index] = s
    return s


@dataclasses.dataclass
class PinnedCsr:
    """A host CSR whose arrays are pinned torch tensors."""
    num_rows: int
    num_cols: int
    row_offsets: "object"  # torch.int64 [num_rows+1], pinned
    col_indices: "object"  # torch.int32, pinned
    values: "object"       # torch.float64, pinned
    sorted_rows: bool = False

    @staticmethod
    def from_csr(a: CsrMatrix) -> "PinnedCsr":
        import torch

        def pin(x, dt):
            return torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).pin_memory()
        base = int(a.row_offsets[0]) if len(a.row_offsets) else 0
        n = a.nnz()
        return PinnedCsr(a.num_rows, a.num_cols, pin(np.asarray(a.row_offsets) - base, np.int64),
                         pin(a.col_indices[base:base + n], np.int32), pin(a.values[base:base + n], np.float64),
                         a.sorted_rows)

    def nnz(self) -> int:
        return int(self.row_offsets[-1]) if self.row_offsets.numel() else 0

    def nbytes(self) -> int:
        return self.row_offsets.numel() * 8 + self.col_indices.numel() * 4 + self.values.numel() * 8


@dataclasses.dataclass
class HostResult:
    """C in pinned host memory; `c` holds numpy views of the pinned tensors."""
    c: CsrMatrix
    h2d_bytes: int
    d2h_bytes: int
    blocks: int
    _keep: Tuple = ()


def _row_cuts(row_offsets: np.ndarray, lo: int, hi: int, blocks: int) -> List[int]:
    """Row cut points of [lo, hi) balancing A's entries (a flop proxy that
    needs no device pass)."""
    if blocks <= 1 or hi - lo <= blocks:
        return [lo, hi]
    ro = row_offsets[lo:hi + 1]
    targets = ro[0] + (ro[-1] - ro[0]) * np.arange(1, blocks) / blocks
    inner = (np.searchsorted(ro, targets) + lo).tolist()
    cuts = [lo] + [int(x) for x in inner] + [hi]
    return sorted(set(cuts))


def multiply_host(a: PinnedCsr, b: Optional[PinnedCsr] = None, cfg: Optional[SpgemmConfig] = None,
                  a_rows: Optional[Tuple[int, int]] = None, blocks: Optional[int] = None,
                  device=None, out: Optional[Tuple] = None, timeline: Optional[list] = None) -> HostResult:
    """C = A*B from pinned host CSR to pinned host CSR.

    b None (or b is a): C = A*A, uploaded once.  a_rows=(lo, hi): A is rows
    [lo, hi) of B (a is ignored then), so only B is uploaded.  out = pinned
    (row_offsets int64, col_indices int32, values float64) tensors to fill
    when large enough (else C's arrays come from torch's pinned cache).
    timeline: a list that receives (label, cuda event) marks."""
    import torch

    def mark(label, stream):
        if timeline is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            timeline.append((label, ev))
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    main = torch.cuda.current_stream(dev)
    side = _copy_stream(dev)
    same = b is None or b is a
    src_b = a if same else b
    if a_rows is not None:
        same = True
        src_b = b if b is not None else a
    lo, hi = a_rows if a_rows is not None else (0, (a if a is not None else src_b).num_rows)

    # ---- uploads: structure on the main stream, values on the copy stream ----
    def up_structure(x: PinnedCsr):
        return (x.row_offsets.to(dev, non_blocking=True), x.col_indices.to(dev, non_blocking=True))

    mark("start", main)
    b_ro_host = src_b.row_offsets.numpy()
    band = None
    if a_rows is not None and (lo, hi) != (0, src_b.num_rows) and hi > lo:
        # A is rows [lo, hi) of B: only the B rows those rows reference (their
        # column band, plus A's own rows) need to travel
        acols = src_b.col_indices.numpy()[b_ro_host[lo]:b_ro_host[hi]]
        if acols.size:
            r0 = min(lo, int(acols.min()))
            r1 = max(hi, int(acols.max()) + 1)
            band = (r0, r1)
    chunk_rows, chunk_events = [], []  # B's values in row chunks (C = A*A path)
    if band is None:
        ro_b, ci_b = up_structure(src_b)
        side.wait_stream(main)
        if same and src_b.nnz() >= (1 << 22):
            # values in 8 row chunks, each with an event: a block of C waits
            # only for the B rows it references
            v_b = torch.empty(max(src_b.nnz(), 1), dtype=torch.float64, device=dev)
            bc = _row_cuts(b_ro_host, 0, src_b.num_rows, 8)
            with torch.cuda.stream(side):
                for c0, c1 in zip(bc[:-1], bc[1:]):
                    q0, q1 = int(b_ro_host[c0]), int(b_ro_host[c1])
                    if q1 > q0:
                        v_b[q0:q1].copy_(src_b.values[q0:q1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(side)
                    chunk_rows.append(c1)
                    chunk_events.append(ev)
        else:
            with torch.cuda.stream(side):
                v_b = src_b.values.to(dev, non_blocking=True)
        h2d = src_b.nbytes()
    else:
        # full row offsets; columns/values of the band rows at their own offsets
        q0, q1 = int(b_ro_host[band[0]]), int(b_ro_host[band[1]])
        ro_b = src_b.row_offsets.to(dev, non_blocking=True)
        ci_b = torch.empty(max(src_b.nnz(), 1), dtype=torch.int32, device=dev)
        v_b = torch.empty(max(src_b.nnz(), 1), dtype=torch.float64, device=dev)
        ci_b[q0:q1].copy_(src_b.col_indices[q0:q1], non_blocking=True)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            v_b[q0:q1].copy_(src_b.values[q0:q1], non_blocking=True)
        h2d = src_b.row_offsets.numel() * 8 + (q1 - q0) * 12
    mark("structure uploaded", main)
    if not same:
        ro_a, ci_a = up_structure(a)
        with torch.cuda.stream(side):
            v_a = a.values.to(dev, non_blocking=True)
        h2d += a.nbytes()
    values_ready = torch.cuda.Event()
    values_ready.record(side)
    mark("values uploaded", side)
    dB = DeviceCsr(src_b.num_rows, src_b.num_cols, ro_b, ci_b, v_b, src_b.sorted_rows, src_b.nnz())
    if same:
        dA_full, a_host_ro = dB, src_b.row_offsets.numpy()
    else:
        dA_full = DeviceCsr(a.num_rows, a.num_cols, ro_a, ci_a, v_a, a.sorted_rows, a.nnz())
        a_host_ro = a.row_offsets.numpy()

    nnz_a = int(a_host_ro[hi] - a_host_ro[lo])
    if blocks is None:
        blocks = 1 if nnz_a < (1 << 22) else 8
    cuts = _row_cuts(a_host_ro, lo, hi, blocks)
    # the last B row each block of A references (its own rows included): the
    # value chunk it waits for
    need_row = None
    if chunk_events:
        tops = []
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            q0, q1 = int(a_host_ro[r0]), int(a_host_ro[r1])
            tops.append(ci_b[q0:q1].max() if q1 > q0 else torch.zeros((), dtype=torch.int32, device=dev))
        need_row = [max(int(t), r1 - 1) for t, r1 in zip(torch.stack(tops).cpu().tolist(), cuts[1:])]

    # ---- one symbolic over A's structure (overlaps the value upload) ----
    dA = dA_full.row_block(lo, hi)
    h = symbolic(dA, dB, cfg, stream=main)
    nnz_c = h.nnz_c()
    m = hi - lo
    c_ro = h.device_row_offsets(main)
    # C's offsets at the block boundaries only (a gather of len(cuts) values,
    # not a pageable copy of all m + 1 offsets)
    bidx = torch.tensor([c - lo for c in cuts], dtype=torch.int64, device=dev)
    ro_cut = dict(zip((c - lo for c in cuts), c_ro.index_select(0, bidx).cpu().tolist()))
    mark("symbolic done", main)
    if out is not None and out[0].numel() >= m + 1 and out[1].numel() >= nnz_c and out[2].numel() >= nnz_c:
        o_ro, o_ci, o_v = out
    else:
        o_ro = torch.empty(m + 1, dtype=torch.int64, pin_memory=True)
        o_ci = torch.empty(max(nnz_c, 1), dtype=torch.int32, pin_memory=True)
        o_v = torch.empty(max(nnz_c, 1), dtype=torch.float64, pin_memory=True)
    d_ci = torch.empty(max(nnz_c, 1), dtype=torch.int32, device=dev)
    d_v = torch.empty(max(nnz_c, 1), dtype=torch.float64, device=dev)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        o_ro[:m + 1].copy_(c_ro, non_blocking=True)

    # ---- numeric per row block; block k's C copies out while block k+1 computes ----
    if need_row is None:
        main.wait_event(values_ready)
    for k, (r0, r1) in enumerate(zip(cuts[:-1], cuts[1:])):
        if need_row is not None:
            c = next(q for q, e in enumerate(chunk_rows) if e > need_row[k])
            main.wait_event(chunk_events[c])
        b0, b1 = r0 - lo, r1 - lo
        numeric_rows(dA, dB, h, b0, b1, d_ci, d_v, stream=main)
        done = torch.cuda.Event()
        done.record(main)
        side.wait_event(done)
        e0, e1 = ro_cut[b0], ro_cut[b1]
        if e1 > e0:
            with torch.cuda.stream(side):
                o_ci[e0:e1].copy_(d_ci[e0:e1], non_blocking=True)
                o_v[e0:e1].copy_(d_v[e0:e1], non_blocking=True)
        mark(f"numeric {r0}:{r1}", main)
        mark(f"copied {r0}:{r1}", side)
    main.wait_stream(side)
    main.synchronize()  # the reference's multiply returns a finished host CSR
    # a device error raised by any block (row overflow/short, pool or bucket
    # overflow) surfaces here as the reference's logic_error would
    h.check()
    sorted_c = bool(cfg.sort_output) if cfg is not None else False
    c = CsrMatrix(m, src_b.num_cols, o_ro.numpy()[:m + 1], o_ci.numpy()[:nnz_c], o_v.numpy()[:nnz_c], sorted_c)
    d2h = (m + 1) * 8 + nnz_c * 12
    return HostResult(c, h2d, d2h, len(cuts) - 1, (o_ro, o_ci, o_v))
