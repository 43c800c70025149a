"""CPU: the multi-GPU host logic (paper_1801_03065_b200/shard.py) — flop-balanced
cut points, B broadcast, nnz all-gather and C block offsets — at world size 2
over gloo.  The per-rank compute is injected (the oracle) because there is no
GPU here; on a B200 box the same code runs over NCCL with the CUDA engine."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1801_03065_b200 import shard


def test_flop_cut_points_balance():
    rng = np.random.default_rng(0)
    f = rng.integers(0, 1000, 10_000)
    cum = np.cumsum(f)
    for parts in (1, 2, 4, 8):
        cuts = shard.flop_cut_points(cum, parts)
        assert cuts[0] == 0 and cuts[-1] == len(f) and len(cuts) == parts + 1
        assert all(x <= y for x, y in zip(cuts, cuts[1:]))
        per = [f[cuts[g]:cuts[g + 1]].sum() for g in range(parts)]
        assert max(per) - min(per) <= 2 * f.max()  # balanced to within one row
        tcuts = shard.flop_cut_points(torch.from_numpy(cum), parts)
        assert tcuts == cuts


def test_flop_cut_points_skewed_and_empty():
    f = np.array([0, 0, 100, 0, 1, 1, 1, 1])
    cuts = shard.flop_cut_points(np.cumsum(f), 2)
    assert cuts == [0, 3, 8]
    assert shard.flop_cut_points(np.zeros(0, np.int64), 4) == [0, 0, 0, 0, 0]


def test_block_offsets():
    assert shard.block_offsets([3, 0, 5]) == [0, 3, 3, 8]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_compute(block, b):
    from oracle.oracle import Oracle
    import paper_1801_03065_b200 as kk
    o = Oracle()
    ah, bh = block.to_host(), b.to_host()
    ro, cols, vals = o.multiply(ah, bh)
    _, fl, _ = o.flops_stats(ah, bh)
    c = kk.DeviceCsr(ah.num_rows, bh.num_cols, torch.from_numpy(ro), torch.from_numpy(cols.copy()),
                     torch.from_numpy(vals.copy()), False, int(ro[-1]))
    return c, None, fl


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1801_03065_b200 as kk
    from paper_1801_03065_b200 import generators as G
    from oracle.oracle import Oracle
    a = G.laplace3d(9)
    da = kk.DeviceCsr(a.num_rows, a.num_cols, torch.from_numpy(a.row_offsets), torch.from_numpy(a.col_indices),
                      torch.from_numpy(a.values), True, a.nnz())
    # B lives on rank 0 only and is broadcast
    db = shard.broadcast_csr(da if rank == 0 else None, 0, rank, "cpu")
    per_row, _, _ = Oracle().flops_stats(a, a)
    cuts = shard.flop_cut_points(np.cumsum(per_row), world)
    s = shard.sharded_multiply(da, db, rank, world, cuts=cuts, compute=_cpu_compute)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), lo=s.lo, hi=s.hi, base=s.base, total=s.nnz_total,
             ro=s.c.row_offsets.numpy(), ci=s.c.col_indices.numpy(), v=s.c.values.numpy(), fl=s.flops_local)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_multiply(tmp_path, oracle):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from paper_1801_03065_b200 import generators as G
    a = G.laplace3d(9)
    ro, cols, vals = oracle.multiply(a, a)
    blocks = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    assert blocks[0]["lo"] == 0 and blocks[-1]["hi"] == a.num_rows
    assert blocks[0]["hi"] == blocks[1]["lo"]
    total = 0
    for b in blocks:
        lo, hi, base = int(b["lo"]), int(b["hi"]), int(b["base"])
        assert base == ro[lo]  # all-gathered block offset == global row offset
        assert np.array_equal(b["ro"] + base, ro[lo:hi + 1])
        assert np.array_equal(b["ci"], cols[ro[lo]:ro[hi]])
        assert np.array_equal(b["v"].view(np.int64), vals[ro[lo]:ro[hi]].view(np.int64))
        assert int(b["total"]) == ro[-1]
        total += int(b["fl"])
    _, fl, _ = oracle.flops_stats(a, a)
    assert total == fl
    # flop balance: the two halves differ by at most one row's flops
    assert abs(int(blocks[0]["fl"]) - int(blocks[1]["fl"])) <= 729


def _band_worker(rank, world, port, outdir, kind):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1801_03065_b200 as kk
    from paper_1801_03065_b200 import generators as G
    from oracle.oracle import Oracle
    a = G.laplace3d(9) if kind == "stencil" else G.rmat(8, 8, 3)
    da = kk.DeviceCsr(a.num_rows, a.num_cols, torch.from_numpy(a.row_offsets), torch.from_numpy(a.col_indices),
                      torch.from_numpy(a.values), True, a.nnz())
    per_row, _, _ = Oracle().flops_stats(a, a)
    cuts = shard.flop_cut_points(np.cumsum(per_row), world)
    lo, hi = cuts[rank], cuts[rank + 1]
    own = shard.own_rows(da, lo, hi)  # the only rows of B = A this rank holds
    out = {}
    for mode in ("band", "all"):
        need = shard.column_band(da, lo, hi) if mode == "band" else (0, a.num_rows)
        band, nbytes = shard.exchange_band(own, cuts, need, rank, world, a.num_rows, a.num_cols)
        s = shard.sharded_multiply(band, band, rank, world, cuts=cuts, compute=_cpu_compute)
        out[mode] = dict(lo=s.lo, hi=s.hi, base=s.base, ro=s.c.row_offsets.numpy(), ci=s.c.col_indices.numpy(),
                         v=s.c.values.numpy(), need0=need[0], need1=need[1], nbytes=nbytes,
                         band_nnz=band.nnz())
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **{f"{m}_{k}": v for m, d in out.items() for k, v in d.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "stencil"), (3, "stencil"), (3, "rmat")])
def test_gloo_band_exchange(tmp_path, oracle, world, kind):
    """B distributed by row blocks (each rank holds only its own rows of B = A):
    the band exchange delivers exactly the rows a block references — the halo
    for a stencil — and with the whole range requested it is an all-gatherv.
    The assembled C blocks equal the single-process product bit for bit."""
    mp.spawn(_band_worker, args=(world, _free_port(), str(tmp_path), kind), nprocs=world, join=True)
    from paper_1801_03065_b200 import generators as G
    a = G.laplace3d(9) if kind == "stencil" else G.rmat(8, 8, 3)
    ro, cols, vals = oracle.multiply(a, a)
    blocks = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    for mode in ("band", "all"):
        for b in blocks:
            lo, hi, base = int(b[f"{mode}_lo"]), int(b[f"{mode}_hi"]), int(b[f"{mode}_base"])
            assert base == ro[lo]
            assert np.array_equal(b[f"{mode}_ro"] + base, ro[lo:hi + 1])
            assert np.array_equal(b[f"{mode}_ci"], cols[ro[lo]:ro[hi]])
            assert np.array_equal(b[f"{mode}_v"].view(np.int64), vals[ro[lo]:ro[hi]].view(np.int64))
    if kind == "stencil":
        n = 9
        halo = n * n + n + 1
        for r, b in enumerate(blocks):
            lo, hi = int(b["band_lo"]), int(b["band_hi"])
            # the band of a 27-point stencil block is at most the block plus one
            # plane, one line and one point on each side
            assert max(0, lo - halo) <= int(b["band_need0"]) <= lo
            assert hi <= int(b["band_need1"]) <= min(n ** 3, hi + halo)
            assert int(b["all_band_nnz"]) == a.nnz()
            assert 0 < int(b["band_nbytes"]) < int(b["all_nbytes"])
