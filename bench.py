"""Benchmark: kkSpGEMM on B200 — BASELINE.json metric on config 2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config 2] [--scale 1.0] [--broadcast]

A step is one full NoReuse multiply (symbolic + numeric, cli.cpp:137-151) of
C = A*A, A = 3D 27-point Laplacian 160^3 (BASELINE configs[1]), fp64, inputs
resident in HBM.  `value` is whole-job GFLOP/s = 2*flops/t (cli.cpp:124-128);
the numeric-only (structure reuse) rate is reported beside it.  Under torchrun
(N>1) rows of C are split into flop-balanced blocks, one per rank;
B is resident on every rank (or broadcast over NCCL each step with
--broadcast); time is the max over ranks of CUDA-event spans.

Only the cpu_baseline leg and `--impl reference` execute the reference
(oracle/_ref, compiled from its own sources) — as the measured CPU baseline,
never on the GPU path.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "GFLOP/s"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


def workload(cfg: int, scale: float):
    from paper_1801_03065_b200 import generators as G
    if cfg == 1:
        n = int(1000 * scale)
        return G.laplace2d(n), f"c1: C=A*A, 2D 5-point Laplacian {n}^2, fp64"
    if cfg == 2:
        n = int(160 * scale)
        return G.laplace3d(n), f"c2: C=A*A, 3D 27-point Laplacian {n}^3, fp64"
    if cfg == 4:
        return G.rmat(20, 16, 1), "c4: C=A*A, R-MAT scale 20 ef 16, fp64"
    if cfg == 5:
        n = int(200 * scale)
        return G.laplace3d(n), f"c5: C=A*A, 3D 27-point Laplacian {n}^3, fp64"
    raise SystemExit(f"config {cfg} is a parity-test case, not a bench line")


def row_sample(a, every: int):
    """Rows 0, every, 2*every, ... of A (rows of C are independent)."""
    from paper_1801_03065_b200 import CsrMatrix
    rows = np.arange(0, a.num_rows, every)
    lo, hi = a.row_offsets[rows], a.row_offsets[rows + 1]
    lens = hi - lo
    ro = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(lens, out=ro[1:])
    idx = np.concatenate([np.arange(l, h) for l, h in zip(lo, hi)]) if len(rows) else np.zeros(0, np.int64)
    return CsrMatrix(len(rows), a.num_cols, ro, a.col_indices[idx], a.values[idx], True)


def cpu_reference_sampler(a, budget_s: float = 12.0, min_every: int = 4):
    """Size a row sample of the workload so one reference multiply (oracle/_ref,
    all host threads) takes about budget_s/3.  Returns (run, flops, cores, kind,
    every): run() times one NoReuse multiply of the sample in seconds."""
    cores = os.cpu_count() or 1
    from oracle.oracle import Oracle, Reference, reference_available
    o = Oracle()
    if reference_available():
        ref, kind = Reference(), "reference"
    else:
        ref, kind = None, "port"

    def run_on(s):
        if ref is not None:
            ms, _ = ref.multiply_ms(s, a, worker_count=cores)
            return ms / 1e3
        t0 = time.perf_counter()
        o.multiply(s, a)
        return time.perf_counter() - t0

    every = 256
    while True:
        s = row_sample(a, every)
        _, fl, _ = o.flops_stats(s, a)
        t = run_on(s)
        if t > budget_s / 3 or every <= min_every:
            break
        every = max(min_every, every // 4)
    return (lambda: run_on(s)), fl, (cores if ref else 1), kind, every, s.num_rows


def cpu_reference_rate(a, budget_s: float = 12.0, min_every: int = 4):
    """The reference's multiply on a row sample: mean of three timed runs.
    Returns (gflops, cores, kind, sample)."""
    run, fl, cores, kind, every, rows = cpu_reference_sampler(a, budget_s, min_every)
    times = [run() for _ in range(3)]
    tm = statistics.mean(times)
    sample = (f"rows 0::{every} of A ({rows} rows, {fl} mults) times full B; mean of "
              f"{len(times)} NoReuse multiplies, worker_count={cores}")
    return 2.0 * fl / tm / 1e9, cores, kind, sample


class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.p is None:
            return
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=5)
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_bytes_numeric(m, nnz_a, flops, nnz_c):
    # SURVEY.md §8d Gustavson traffic model
    return 16 * (m + 1) + 28 * nnz_a + 12 * flops + 12 * nnz_c


def load_traffic(name: str):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p)).get(name)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kk", choices=["kk", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--broadcast", action="store_true", help="broadcast B over NCCL every step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    a_host, wl = workload(args.config, args.scale)

    if args.impl == "reference":
        if rank != 0:
            return
        # each step: one NoReuse multiply of a row sample sized to ~4 s
        run, sfl, cores, kind, every, rows = cpu_reference_sampler(a_host)
        for _ in range(args.warmup):
            run()
        times = [run() for _ in range(args.steps)]
        rate = 2.0 * sfl * len(times) / sum(times) / 1e9
        sample = (f"rows 0::{every} of A ({rows} rows, {sfl} mults) times full B per step; "
                  f"{args.steps} timed + {args.warmup} warm-up NoReuse multiplies, worker_count={cores}")
        from oracle.oracle import Oracle
        _, fl, _ = Oracle().flops_stats(a_host, a_host)
        line = {"metric": METRIC, "value": rate, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 2.0 * fl / rate / 1e6,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": wl, "mode": "symbolic+numeric (NoReuse)"},
                "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
                "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    import paper_1801_03065_b200 as kk

    # one process per GPU over NCCL; KK_BENCH_BACKEND=gloo (with KK_BENCH_SAME_GPU=1)
    # runs the multi-rank code path on a single GPU as a smoke test (host
    # collectives only: no rank's kernel waits on another's)
    backend = os.environ.get("KK_BENCH_BACKEND", "nccl")
    if os.environ.get("KK_BENCH_SAME_GPU"):
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    A = a_host.to_device(dev)
    B = A  # C = A*A
    nnz_a = a_host.nnz()
    m = a_host.num_rows

    # ---- flop-balanced row partition, not timed ----
    from paper_1801_03065_b200 import shard
    lo, hi = 0, m
    if world > 1:
        cuts = shard.flop_cut_points(torch.cumsum(kk.row_flops(A, B), 0), world)
        lo, hi = cuts[rank], cuts[rank + 1]
    A_shard = A.row_block(lo, hi)

    # ---- warm-up and one reference multiply for counts ----
    h0 = kk.symbolic(A_shard, B)
    info = h0._info()
    flops_local = int(info.flops.total_flops)
    nnz_c_local = int(info.nnz_c)
    cols = torch.empty(max(nnz_c_local, 1), dtype=torch.int32, device=dev)
    vals = torch.empty(max(nnz_c_local, 1), dtype=torch.float64, device=dev)

    def bcast_b(values_only: bool = False):
        # B broadcast over NCCL from rank 0 every step (the "with broadcast"
        # timing); numeric-only passes re-send only B's values (SURVEY §8e:
        # the structure is unchanged under reuse)
        if world > 1 and args.broadcast:
            for t in ((B.values,) if values_only else (B.row_offsets, B.col_indices, B.values)):
                dist.broadcast(t, src=0)  # in place: ranks > 0 compute on it

    def step_symnum():
        # the reference's multiply: flops/gate, compression, symbolic, scan,
        # C allocation (torch's caching allocator) and numeric
        bcast_b()
        h = kk.symbolic(A_shard, B)
        return kk.numeric(A_shard, B, h)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step_symnum()
    barrier()

    l0 = kk.kernel_launch_count()
    with Clocks(local) as clk:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step_symnum()
        ev1.record(stream)
        barrier()
    launches = kk.kernel_launch_count() - l0
    ms_local = ev0.elapsed_time(ev1)

    # ---- numeric-only (structure reuse): one symbolic, K numerics ----
    # h0 replays the slot map recorded on its second pass (kk_replay.cu) when
    # eligible; h_hash is held on the hashing kernels (KK_NO_REPLAY at plan
    # time) so both numeric paths are timed on the same operands
    os.environ["KK_NO_REPLAY"] = "1"
    h_hash = kk.symbolic(A_shard, B)
    del os.environ["KK_NO_REPLAY"]

    def time_numeric(h):
        for _ in range(max(args.warmup, 2)):
            kk.numeric(A_shard, B, h, out=(cols, vals))
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            bcast_b(values_only=True)
            kk.numeric(A_shard, B, h, out=(cols, vals))
        e1.record(stream)
        barrier()
        return e0.elapsed_time(e1)

    ms_num_local = time_numeric(h0)
    replay_state = h0.replay_state
    ms_hash_local = time_numeric(h_hash) if replay_state == 2 else ms_num_local
    num_kernel_ms = ms_hash_local / args.steps  # one row-kernel launch per numeric (single class)
    replay_ms = ms_num_local / args.steps

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    ms = allmax(ms_local) / args.steps
    ms_num = allmax(ms_num_local) / args.steps
    ms_hash = allmax(ms_hash_local) / args.steps
    # symbolic phase inside the NoReuse step = step - numeric (hashing kernels, the
    # numeric a NoReuse multiply runs); its roofline uses SURVEY §8d bytes_sym
    ms_sym = max(ms - ms_hash, 1e-6)
    flops = allsum(flops_local)
    nnz_c = allsum(nnz_c_local)
    value = 2.0 * flops / (ms / 1e3) / 1e9
    value_num = 2.0 * flops / (ms_num / 1e3) / 1e9

    # ---- end to end through the public API with host buffers (rank-local) ----
    # host.multiply_host: pinned host CSR in, pinned host C out; A = rows
    # [lo, hi) of B = A, so B is the only upload; C's row blocks are copied
    # out while later blocks compute
    e2e = None
    if not args.no_e2e:
        from paper_1801_03065_b200 import host
        pa = host.PinnedCsr.from_csr(a_host)
        outbuf = (torch.empty(hi - lo + 1, dtype=torch.int64).pin_memory(),
                  torch.empty(max(nnz_c_local, 1), dtype=torch.int32).pin_memory(),
                  torch.empty(max(nnz_c_local, 1), dtype=torch.float64).pin_memory())

        def e2e_step():
            return host.multiply_host(None, pa, a_rows=(lo, hi), out=outbuf)

        r = e2e_step()
        assert r.c.nnz() == nnz_c_local
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        ksteps = max(1, min(args.steps, 5))
        t0.record(stream)
        for _ in range(ksteps):
            r = e2e_step()
        t1.record(stream)
        barrier()
        ms_e2e = allmax(t0.elapsed_time(t1)) / ksteps
        e2e = {"value": 2.0 * flops / (ms_e2e / 1e3) / 1e9, "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": int(allsum(r.h2d_bytes)), "d2h_bytes_per_step": int(allsum(r.d2h_bytes)),
               "row_blocks": r.blocks,
               "path": "host.multiply_host (C ABI): pinned host CSR in, pinned host C out, copy/compute overlap"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks, peak_kind = _peaks()
    full_size = args.scale == 1.0 and world == 1  # the committed ncu traffic is for this workload
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    bytes_num = algorithmic_bytes_numeric(hi - lo, nnz_a if world == 1 else info.nnz_a, flops_local, nnz_c_local)
    achieved = bytes_num / (num_kernel_ms / 1e3) / 1e9
    # flops/gate pass, compress B, union over (csi, cs) pairs
    n_b = B.num_rows
    if info.compression.applied:
        sym_bytes = (24 * (hi - lo + 1) + 44 * info.nnz_a + 16 * (n_b + 1) + 4 * info.nnz_b
                     + 8 * info.compressed_nnz_b + 8 * info.compression.compressed_flops)
    else:
        sym_bytes = 24 * (hi - lo + 1) + 44 * info.nnz_a + 4 * flops_local
    w = 1 if info.max_row_size <= 256 else 2
    replay_bytes = (24 * (hi - lo + 1) + 28 * (nnz_a if world == 1 else info.nnz_a) + (8 + w) * flops_local
                    + 16 * nnz_c_local)
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        rate, cores, kind, sample = cpu_reference_rate(a_host)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl, "mode": "symbolic+numeric (NoReuse multiply per step)",
                   "m": m, "nnz_a": nnz_a, "flops": int(flops), "nnz_c": int(nnz_c),
                   "parallelism": f"row-shard x{world}" + (f" + {backend} broadcast of B" if args.broadcast else
                                                            " (B resident)"),
                   "l2_policy": "inputs larger than L2 (A = %.2f GB > 126 MB)" % (nnz_a * 12 / 1e9)},
        "numeric_only": {"value": value_num, "unit": UNIT, "ms_per_step": ms_num,
                         "path": "slot replay (kk_replay.cu)" if replay_state == 2 else "hashing kernels",
                         "hashing_kernels": {"value": 2.0 * flops / (ms_hash / 1e3) / 1e9, "unit": UNIT,
                                             "ms_per_step": ms_hash}},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm,
                     "traffic": load_traffic(f"c{args.config}_numeric") if full_size else None,
                     "kernel": "numeric_lp_seq_kernel (numeric phase)", "peak_kind": peak_kind,
                     "algorithmic_bytes": bytes_num,
                     "model": "16(m+1)+28nnzA+12flops+12nnzC (SURVEY §8d)"},
        "roofline_symbolic": {
            "bound": "hbm", "achieved": sym_bytes / (ms_sym / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": sym_bytes / (ms_sym / 1e3) / 1e9 / hbm, "ms_per_step": ms_sym, "algorithmic_bytes": sym_bytes,
            "kernel": "symbolic phase (compress, flops, union, scan) = NoReuse step - hashing numeric",
            "model": "24(m+1)+44nnzA+16(n+1)+4nnzB+8nnzBc+8cflops (compressed; SURVEY §8d)"},
        "roofline_replay": None if replay_state != 2 else {
            "bound": "hbm", "achieved": replay_bytes / (replay_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": replay_bytes / (replay_ms / 1e3) / 1e9 / hbm, "kernel": "replay_numeric_kernel (+ structure fingerprint pass)",
            "traffic": load_traffic(f"c{args.config}_replay") if full_size else None,
            "algorithmic_bytes": replay_bytes, "model": "24(m+1)+28nnzA+(8+w)flops+16nnzC, w = slot bytes"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
