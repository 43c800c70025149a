"""Multi-GPU row sharding of C = A*B.

Rows of C are independent (Alg. 3 is row-private), so the
multiply shards without any data-path collective:

1. per-row flops on the device (``spg_row_flops``), inclusive scan, and G cut
   points at ``total*g/G`` (lower_bound) -> contiguous flop-balanced row blocks;
2. every rank runs symbolic + numeric on its row-block *view* of A against the
   full B — B either resident on every rank or broadcast from ``src`` over
   NCCL (``broadcast_csr``; the only bulk transfer);
3. one 8-byte all-gather of the local nnz gives each C block its base offset
   (exclusive scan); C stays distributed as (local row offsets, base, cols, vals).

The functions take a torch.distributed process group, so the same code runs
over NCCL (one process per GPU) and over gloo on CPU for the host-logic tests
(tests/test_shard.py), where the per-rank compute is injected.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional, Sequence

import numpy as np


def flop_cut_points(cum_flops, parts: int) -> list:
    """Row boundaries [0, r1, ..., m] of `parts` contiguous blocks with
    ~equal flops.  cum_flops is the inclusive prefix sum of per-row flops
    (numpy or torch, length m).  r_g = lower_bound(cum, total*g/parts)."""
    m = len(cum_flops)
    if m == 0:
        return [0] * (parts + 1)
    try:
        import torch
        is_torch = isinstance(cum_flops, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_torch = False
    total = int(cum_flops[-1].item() if is_torch else cum_flops[-1])
    cuts = [0]
    for g in range(1, parts):
        target = total * g // parts
        if is_torch:
            import torch
            r = int(torch.searchsorted(cum_flops, torch.tensor([target], dtype=cum_flops.dtype,
                                                                device=cum_flops.device)).item())
        else:
            r = int(np.searchsorted(cum_flops, target, side="left"))
        cuts.append(max(cuts[-1], min(r + 1 if total > 0 else r, m)))
    cuts.append(m)
    return cuts


def block_offsets(local_nnz: Sequence[int]) -> list:
    """Exclusive scan of the ranks' nnz: base offset of each C block."""
    out, acc = [], 0
    for n in local_nnz:
        out.append(acc)
        acc += int(n)
    return out + [acc]


def broadcast_csr(mat, src: int, rank: int, device, group=None, dist=None):
    """Broadcast a CSR (row offsets, cols, vals) from rank `src`; the other
    ranks allocate and receive.  Returns a kk.DeviceCsr-like object with
    torch tensors on `device` (CPU for gloo)."""
    import torch
    if dist is None:
        import torch.distributed as dist
    from . import DeviceCsr
    shape = torch.zeros(3, dtype=torch.int64, device=device)
    if rank == src:
        shape[0], shape[1], shape[2] = mat.num_rows, mat.num_cols, int(mat.nnz())
    dist.broadcast(shape, src=src, group=group)
    nr, nc, nnz = (int(x) for x in shape.tolist())
    if rank == src:
        ro, ci, v = mat.row_offsets, mat.col_indices, mat.values
    else:
        ro = torch.empty(nr + 1, dtype=torch.int64, device=device)
        ci = torch.empty(nnz, dtype=torch.int32, device=device)
        v = torch.empty(nnz, dtype=torch.float64, device=device)
    for t in (ro, ci, v):
        dist.broadcast(t, src=src, group=group)
    return DeviceCsr(nr, nc, ro, ci, v, True, nnz)


@dataclasses.dataclass
class Shard:
    rank: int
    world: int
    lo: int                 # first row of the block
    hi: int                 # one past the last row
    c: object               # local C block (row offsets relative to the block)
    nnz_local: int
    base: int               # global offset of the block's first entry
    nnz_total: int
    flops_local: int
    handle: object = None


def sharded_multiply(a, b, rank: int, world: int, group=None, cuts: Optional[list] = None,
                     compute: Optional[Callable] = None, dist=None, cfg=None) -> Shard:
    """This rank's block of C = A*B.  `a`, `b`: kk.DeviceCsr (full A visible,
    full B resident on this rank).  `compute(a_block, b)` -> (c, handle,
    flops_local); defaults to the GPU engine."""
    import torch
    if dist is None:
        import torch.distributed as dist
    from . import multiply, row_flops
    if cuts is None:
        per_row = row_flops(a, b)
        cuts = flop_cut_points(torch.cumsum(per_row, 0), world)
    lo, hi = cuts[rank], cuts[rank + 1]
    block = a.row_block(lo, hi)
    if compute is None:
        res = multiply(block, b, cfg)
        c, handle, flops_local = res.c, res.handle, res.handle.flops.total_flops
    else:
        c, handle, flops_local = compute(block, b)
    nnz_local = int(c.nnz())
    dev = c.row_offsets.device if hasattr(c.row_offsets, "device") else "cpu"
    mine = torch.tensor([nnz_local], dtype=torch.int64, device=dev)
    allv = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    if world > 1:
        dist.all_gather(allv, mine, group=group)
    else:
        allv = [mine]
    offs = block_offsets([int(t.item()) for t in allv])
    return Shard(rank, world, lo, hi, c, nnz_local, offs[rank], offs[-1], int(flops_local), handle)


# ---------------------------------------------------------------------------
# B distributed by rows: each rank owns a row block of B and receives only the
# rows its block of A references (the stencil halo; with the
# whole row range requested it is the all-gatherv fallback for a B that is
# not replicated).
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class OwnedRows:
    """Rows [lo, hi) of a CSR held by this rank: row offsets rebased to 0."""
    lo: int
    hi: int
    row_offsets: object  # torch.int64 [hi-lo+1]
    col_indices: object  # torch.int32
    values: object       # torch.float64


def own_rows(b, lo: int, hi: int) -> OwnedRows:
    """This rank's row block of `b` (copied out of a full matrix; in a
    distributed run it is what the rank holds to begin with)."""
    ro = b.row_offsets[lo:hi + 1]
    s, e = int(ro[0].item()), int(ro[-1].item())
    return OwnedRows(lo, hi, (ro - s).clone(), b.col_indices[s:e].clone(), b.values[s:e].clone())


def column_band(a, lo: int, hi: int) -> tuple:
    """[r0, r1): the B rows that rows [lo, hi) of A reference, widened to
    include [lo, hi) itself (for C = A*A the rank's own rows are its A block)."""
    ro = a.row_offsets
    s, e = int(ro[lo].item()), int(ro[hi].item())
    if e <= s:
        return (lo, hi)
    cols = a.col_indices[s:e]
    return (min(lo, int(cols.min().item())), max(hi, int(cols.max().item()) + 1))


def _intersect(a0, a1, b0, b1):
    lo, hi = max(a0, b0), min(a1, b1)
    return (lo, hi) if hi > lo else None


def exchange_band(own: OwnedRows, cuts: Sequence[int], need: tuple, rank: int, world: int,
                  num_rows: int, num_cols: int, group=None, dist=None, needs: Optional[list] = None):
    """Assemble this rank's view of B holding rows [need[0], need[1]).

    Owners are given by `cuts` (rank q owns [cuts[q], cuts[q+1])).  Every
    owner sends each requester the intersection of its rows with the
    requested range: row lengths first, then columns and values (two rounds
    of batched point-to-point transfers, NCCL on GPUs, gloo on CPU).  The
    result is a DeviceCsr of num_rows rows whose row offsets are rebased so
    that rows outside the band are empty; its columns are global.  Returns
    (view, bytes received from other ranks)."""
    import torch
    if dist is None:
        import torch.distributed as dist
    from . import DeviceCsr
    dev = own.row_offsets.device
    if needs is None:
        mine = torch.tensor([need[0], need[1]], dtype=torch.int64, device=dev)
        allv = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(world)]
        if world > 1:
            dist.all_gather(allv, mine, group=group)
        else:
            allv = [mine]
        needs = [tuple(int(x) for x in t.tolist()) for t in allv]
    lens_own = own.row_offsets[1:] - own.row_offsets[:-1]

    # round 1: row lengths of every piece
    pieces = {}   # owner q -> (r0, r1) of the rows this rank receives from q
    ops, recv_lens = [], {}
    for q in range(world):
        got = _intersect(cuts[q], cuts[q + 1], need[0], need[1])
        if got is not None:
            pieces[q] = got
    for q in range(world):
        if q == rank:
            continue
        give = _intersect(own.lo, own.hi, needs[q][0], needs[q][1])
        if give is not None:
            ops.append(dist.P2POp(dist.isend, lens_own[give[0] - own.lo:give[1] - own.lo].contiguous(), q,
                                  group=group))
        if q in pieces:
            r0, r1 = pieces[q]
            recv_lens[q] = torch.empty(r1 - r0, dtype=torch.int64, device=dev)
            ops.append(dist.P2POp(dist.irecv, recv_lens[q], q, group=group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()

    # round 2: columns and values
    ops, recv = [], {}
    nbytes = 0
    for q in range(world):
        if q == rank:
            continue
        give = _intersect(own.lo, own.hi, needs[q][0], needs[q][1])
        if give is not None:
            s = int(own.row_offsets[give[0] - own.lo].item())
            e = int(own.row_offsets[give[1] - own.lo].item())
            ops.append(dist.P2POp(dist.isend, own.col_indices[s:e].contiguous(), q, group=group))
            ops.append(dist.P2POp(dist.isend, own.values[s:e].contiguous(), q, group=group))
        if q in pieces:
            n = int(recv_lens[q].sum().item())
            ci = torch.empty(n, dtype=torch.int32, device=dev)
            v = torch.empty(n, dtype=torch.float64, device=dev)
            recv[q] = (ci, v)
            ops.append(dist.P2POp(dist.irecv, ci, q, group=group))
            ops.append(dist.P2POp(dist.irecv, v, q, group=group))
            nbytes += recv_lens[q].numel() * 8 + n * 12
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()

    # assemble in row order
    lens, cols, vals = [], [], []
    for q in sorted(pieces):
        r0, r1 = pieces[q]
        if q == rank:
            s = int(own.row_offsets[r0 - own.lo].item())
            e = int(own.row_offsets[r1 - own.lo].item())
            lens.append(lens_own[r0 - own.lo:r1 - own.lo])
            cols.append(own.col_indices[s:e])
            vals.append(own.values[s:e])
        else:
            lens.append(recv_lens[q])
            cols.append(recv[q][0])
            vals.append(recv[q][1])
    band_len = torch.cat(lens) if lens else torch.zeros(0, dtype=torch.int64, device=dev)
    ro = torch.zeros(num_rows + 1, dtype=torch.int64, device=dev)
    if band_len.numel():
        ro[need[0] + 1:need[1] + 1] = torch.cumsum(band_len, 0)
        ro[need[1] + 1:] = ro[need[1]]
    ci = torch.cat(cols) if cols else torch.zeros(0, dtype=torch.int32, device=dev)
    v = torch.cat(vals) if vals else torch.zeros(0, dtype=torch.float64, device=dev)
    return DeviceCsr(num_rows, num_cols, ro, ci, v, True, int(ci.numel())), nbytes
