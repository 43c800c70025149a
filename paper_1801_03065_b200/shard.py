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
