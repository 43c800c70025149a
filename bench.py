"""Benchmark: kkSpGEMM on B200 — the BASELINE.json metric on its configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config 1..5] [--scale 1.0]

Default (the driver's line): config 2, C = A*A for the 3D 27-point Laplacian
160^3 (BASELINE configs[1]), fp64.  A step is one full NoReuse multiply
(symbolic + numeric, cli.cpp:137-151) with the inputs resident in HBM;
`value` is whole-job GFLOP/s = 2*flops/t (cli.cpp:124-128) and the
numeric-only (structure reuse) rate is reported beside it.

  --config 1  2D 5-point 1000^2, C = A*A             (step: sym+num; inputs < L2: L2 flushed between steps)
  --config 2  3D 27-point 160^3, C = A*A             (step: sym+num)
  --config 3  R*(A*P), 3D 27-point 128^3, 2x2x2 aggregation P, R = P^T
                                                     (step: both products, sym+num, AP fed back on device)
  --config 4  R-MAT scale 20, edge factor 16, C = A*A (step: sym+num; default SpgemmConfig)
  --config 5  3D 27-point 200^3, 1 symbolic + numeric passes with perturbed values
                                                     (step: one numeric pass; the 100-pass figure beside it)

Every line carries `roofline` (SURVEY §8d algorithmic bytes of the numeric
phase over its measured time, against MEASURED_PEAKS.json), `cpu_baseline`
(the reference library built from /root/reference, oracle/_ref, on this
host's cores, on a bounded row sample) and `e2e` (the same metric through the
host-memory API with host<->device copies in the timed region).

Under torchrun (N > 1) rows of C are split into flop-balanced blocks
(shard.sharded_multiply); `value` is with B resident on every rank,
and the line also times B shipped per step — broadcast from rank 0 over NCCL,
and the band exchange (each rank owns its rows of B = A and receives only the
rows its block references: the stencil halo).  Times are max over ranks of
CUDA-event spans.

`--impl reference` runs the reference's own CPU multiply (oracle/_ref) on the
same config with all host threads, a bounded row sample per step; its inputs
come from oracle/libgen.so, so that process loads no product library.
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
L2_BYTES = 126 * 1024 * 1024

MODES = {
    1: "symbolic+numeric (NoReuse multiply per step)",
    2: "symbolic+numeric (NoReuse multiply per step)",
    3: "symbolic+numeric of A*P then R*(AP) per step (AP fed back on the device)",
    4: "symbolic+numeric (NoReuse multiply per step)",
    5: "one numeric-only pass per step with perturbed values (1 symbolic, then passes)",
}


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def workload(cfg: int, scale: float, gen):
    """(matrices, label) of a BASELINE config from generator set `gen`."""
    mats = gen.config_matrices(cfg, scale)
    if cfg == 1:
        wl = f"c1: C=A*A, 2D 5-point Laplacian {int(1000 * scale)}^2, fp64"
    elif cfg == 2:
        wl = f"c2: C=A*A, 3D 27-point Laplacian {int(160 * scale)}^3, fp64"
    elif cfg == 3:
        wl = f"c3: R*(A*P), 3D 27-point Laplacian {int(128 * scale)}^3, 2x2x2 aggregation P, R=P^T, fp64"
    elif cfg == 4:
        wl = f"c4: C=A*A, R-MAT scale {int(round(20 + np.log2(scale)))} ef 16, fp64"
    else:
        wl = f"c5: C=A*A, 3D 27-point Laplacian {int(200 * scale)}^3, structure reuse, fp64"
    return mats, wl


def operand_a(cfg: int, scale: float = 1.0):
    """(A, label) of a config from the product generators (profiling scripts)."""
    from paper_1801_03065_b200 import generators as G
    mats, wl = workload(cfg, scale, G)
    return mats["A"], wl


def products(cfg: int, mats):
    """The (A, B) pairs one step multiplies."""
    if cfg == 3:
        return [("A", "P"), ("R", "AP")]
    return [("A", "B")]


def config_dict(cfg, wl, counts, world, parallelism, l2_policy):
    """Identical keys for both arms (the driver compares them)."""
    return {"workload": wl, "mode": MODES[cfg], "m": counts["m"], "nnz_a": counts["nnz_a"],
            "flops": counts["flops"], "nnz_c": counts["nnz_c"], "parallelism": parallelism,
            "l2_policy": l2_policy}


def l2_policy(cfg, mats):
    a = mats["A"]
    in_bytes = a.nnz() * 12 + (a.num_rows + 1) * 8
    if cfg != 3 and in_bytes < L2_BYTES:
        return "inputs (%.0f MB) smaller than L2: a 256 MB buffer is written between timed steps" % (in_bytes / 1e6)
    return "inputs larger than L2 (A = %.2f GB > 126 MB)" % (in_bytes / 1e9)


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


def reference_counts(ref, cfg, mats, cores):
    """m, nnz_a, flops, nnz_c of the full workload from the reference itself."""
    out = {"m": 0, "nnz_a": 0, "flops": 0, "nnz_c": 0}
    for an, bn in products(cfg, mats):
        a, b = mats[an], mats[bn]
        h = ref.symbolic(a, b, worker_count=cores)
        info = h.info()
        out["m"] += a.num_rows
        out["nnz_a"] += a.nnz()
        out["flops"] += int(info["total_flops"])
        out["nnz_c"] += int(info["nnz_c"])
        if cfg == 3 and an == "A":
            cols, vals, _ = h.numeric()
            from paper_1801_03065_b200 import CsrMatrix
            mats["AP"] = CsrMatrix(a.num_rows, b.num_cols, h.row_offsets(), cols, vals, False)
    return out


def cpu_reference_sampler(cfg, mats, budget_s: float = 12.0):
    """A bounded sample of the workload timed on the reference library
    (oracle/_ref, all host threads; else the oracle port, 1 thread).
    Returns (run, sample_flops, cores, kind, label): run() times one sample
    step in seconds."""
    from oracle.oracle import Oracle, Reference, reference_available
    cores = os.cpu_count() or 1
    ref = Reference() if reference_available() else None
    kind = "reference" if ref is not None else "port"
    o = Oracle()

    if cfg == 3:
        a, p, r = mats["A"], mats["P"], mats["R"]
        _, f1, _ = o.flops_stats(a, p)
        if "AP" not in mats:
            ro, ci, v = o.multiply(a, p)
            from paper_1801_03065_b200 import CsrMatrix
            mats["AP"] = CsrMatrix(a.num_rows, p.num_cols, ro, ci, v, False)
        _, f2, _ = o.flops_stats(r, mats["AP"])

        def run():
            if ref is not None:
                t = ref.multiply_ms(a, p, worker_count=cores)[0] + ref.multiply_ms(r, mats["AP"], worker_count=cores)[0]
                return t / 1e3
            t0 = time.perf_counter()
            o.multiply(a, p)
            o.multiply(r, mats["AP"])
            return time.perf_counter() - t0
        return run, f1 + f2, cores if ref else 1, kind, "full c3 (multiply(A,P) + multiply(R,AP)) per step"

    a = mats["A"]
    if cfg == 5:
        every = 16
        s = row_sample(a, every)
        _, fl, _ = o.flops_stats(s, a)
        if ref is not None:
            rh = ref.symbolic(s, a, worker_count=cores)
            rh.set_workers(cores)

            def run():
                t0 = time.perf_counter()
                rh.numeric()
                return time.perf_counter() - t0
        else:
            ro = o.symbolic_row_offsets(s, a)

            def run():
                t0 = time.perf_counter()
                o.numeric(s, a, ro)
                return time.perf_counter() - t0
        return run, fl, cores if ref else 1, kind, (f"numeric-only pass of rows 0::{every} of A ({s.num_rows} rows, "
                                                    f"{fl} mults) times full B, symbolic outside the step")

    def run_on(s):
        if ref is not None:
            ms, _ = ref.multiply_ms(s, a, worker_count=cores)
            return ms / 1e3
        t0 = time.perf_counter()
        o.multiply(s, a)
        return time.perf_counter() - t0

    every = 1024
    while True:
        s = row_sample(a, every)
        _, fl, _ = o.flops_stats(s, a)
        t = run_on(s)
        if t > budget_s / 3 or every <= 1:
            break
        every = max(1, every // 4)
    return (lambda: run_on(s)), fl, (cores if ref else 1), kind, (
        (f"NoReuse multiply of rows 0::{every} of A ({s.num_rows} rows, {fl} mults) times full B per step"
         if every > 1 else "the full NoReuse multiply per step"))


def cpu_baseline(cfg, mats, full_flops):
    from oracle.oracle import cpu_model
    run, fl, cores, kind, label = cpu_reference_sampler(cfg, mats)
    times = [run() for _ in range(3)]
    t = statistics.mean(times)
    return {"value": 2.0 * fl / t / 1e9, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": label + f"; mean of {len(times)} steps", "sample_fraction": fl / max(full_flops, 1),
            "ms_per_sample_step": 1e3 * t, "cpu_model": cpu_model(), "nproc": os.cpu_count()}


class Clocks:
    """nvidia-smi clock / throttle-reason samples (100 ms) over the timed
    region.  The sampler is started first and the region begins only once it
    reports (its start-up takes longer than a short timed region); samples
    from the start-up wait are dropped."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.p = None
        self.lines = []
        self.t0 = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append((time.perf_counter(), line))

    def __enter__(self):
        import threading
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            deadline = time.perf_counter() + 5.0
            while not self.lines and time.perf_counter() < deadline:
                time.sleep(0.01)
        except Exception:
            self.p = None
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.p is None:
            return
        time.sleep(0.15)  # one more sample after the region
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            pass
        for t, line in list(self.lines):
            if t < self.t0:
                continue
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


def bytes_num(m, nnz_a, flops, nnz_c):
    """SURVEY.md §8d Gustavson traffic model of one numeric pass."""
    return 16 * (m + 1) + 28 * nnz_a + 12 * flops + 12 * nnz_c


def load_traffic(name: str):
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(name)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args, rank):
    if rank != 0:
        return
    from oracle.oracle import Reference, cpu_model, generators, reference_available
    mats, wl = workload(args.config, args.scale, generators())
    cores = os.cpu_count() or 1
    counts = None
    if reference_available():
        counts = reference_counts(Reference(), args.config, mats, cores)
    run, sfl, cores_used, kind, label = cpu_reference_sampler(args.config, mats)
    for _ in range(args.warmup):
        run()
    times = [run() for _ in range(args.steps)]
    ms = 1e3 * statistics.mean(times)
    rate = 2.0 * sfl / (ms / 1e3) / 1e9
    if counts is None:
        counts = {"m": mats["A"].num_rows, "nnz_a": mats["A"].nnz(), "flops": None, "nnz_c": None}
    frac = sfl / counts["flops"] if counts["flops"] else None
    line = {"metric": METRIC, "value": rate, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, wl, counts, args.gpus,
                                  f"row-shard x{args.gpus}" + " (B resident)", l2_policy(args.config, mats)),
            "sample_fraction": frac,
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores_used, "kind": kind,
                             "sample": label + f"; {args.steps} timed + {args.warmup} warm-up steps",
                             "sample_fraction": frac, "cpu_model": cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
class StepTimer:
    """Sum of per-step CUDA-event spans on `stream`; an optional L2 flush runs
    between steps outside the spans."""

    def __init__(self, stream, flush_bytes=0):
        import torch
        self.stream = stream
        self.flush = torch.empty(flush_bytes // 4, dtype=torch.float32, device=stream.device) if flush_bytes else None

    def run(self, fn, steps):
        import torch
        evs = []
        for _ in range(steps):
            if self.flush is not None:
                self.flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            fn()
            e1.record(self.stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs)


def run_gpu(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_1801_03065_b200 as kk
    from paper_1801_03065_b200 import generators as G
    from paper_1801_03065_b200 import shard

    backend = os.environ.get("KK_BENCH_BACKEND", "nccl")
    if os.environ.get("KK_BENCH_SAME_GPU"):
        local = 0  # multi-rank code path on one GPU (host collectives only; a smoke test)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    cfg = args.config
    mats, wl = workload(cfg, args.scale, G)
    policy = l2_policy(cfg, mats)
    flush = 256 << 20 if "flushed" in policy else 0
    timer = StepTimer(stream, flush)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

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

    extra = {}
    if cfg == 3:
        res = run_c3(args, kk, mats, dev, timer, barrier)
    elif cfg == 5:
        res = run_c5(args, kk, mats, dev, timer, barrier)
    elif world > 1:
        res = run_sharded(args, kk, shard, mats, dev, timer, barrier, rank, world, dist)
    else:
        res = run_aa(args, kk, mats, dev, timer, barrier)

    ms = allmax(res["ms_total"]) / args.steps
    flops = allsum(res["flops"])
    nnz_c = allsum(res["nnz_c"])
    counts = {"m": int(allsum(res["m"])) if world > 1 else res["m"], "nnz_a": res["nnz_a"],
              "flops": int(flops), "nnz_c": int(nnz_c)}
    value = 2.0 * flops / (ms / 1e3) / 1e9
    num_ms = allmax(res["num_ms_total"]) / res["num_steps"]
    e2e = res.get("e2e")
    if e2e and "ms_per_step" in e2e:
        ms_e2e = allmax(e2e["ms_per_step"])
        e2e["value"] = 2.0 * flops / (ms_e2e / 1e3) / 1e9
        e2e["ms_per_step"] = ms_e2e
        e2e["h2d_bytes_per_step"] = int(allsum(e2e["h2d_bytes_per_step"]))
        e2e["d2h_bytes_per_step"] = int(allsum(e2e["d2h_bytes_per_step"]))
    for key in ("with_broadcast", "with_band_exchange"):
        if key in res:
            t = allmax(res[key]["ms_total"]) / args.steps
            extra[key] = {"value": 2.0 * flops / (t / 1e3) / 1e9, "unit": UNIT, "ms_per_step": t,
                          "bytes_per_step": int(allsum(res[key]["bytes"])), "path": res[key]["path"]}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks, peak_kind = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    bnum = res["bytes_num"]
    achieved = bnum / (num_ms / 1e3) / 1e9
    full_size = args.scale == 1.0 and world == 1
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(cfg, mats, counts["flops"])
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, wl, counts, world,
                              f"row-shard x{world} (B resident; B shipped per step timed beside)" if world > 1
                              else "row-shard x1 (B resident)", policy),
        "numeric_only": res["numeric_only"],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": load_traffic(f"c{cfg}_numeric") if full_size else None,
                     "kernel": res["num_kernel"], "peak_kind": peak_kind, "algorithmic_bytes": bnum,
                     "ms_per_launch": num_ms,
                     "model": "16(m+1)+28nnzA+12flops+12nnzC per numeric pass (SURVEY §8d)"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(res["launches"]),
        "clocks": res["clocks"],
    }
    for k in ("roofline_symbolic", "roofline_replay", "detail"):
        if res.get(k) is not None:
            line[k] = res[k]
    line.update(extra)
    print(json.dumps(line), flush=True)
    if args.csv:
        write_records(args.csv, line, res)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def write_records(path, line, res):
    """The line as the reference's BenchRecord rows (bench.cpp:28-102; the
    reference CLI's `bench` output, cli.cpp:132-174): one NoReuse row and one
    reuse (numeric-only) row, GPU columns in the sidecar .gpu.csv."""
    import torch
    from paper_1801_03065_b200 import harness as H
    cfg = line["config"]
    det = res.get("detail") or {}
    base = dict(problem=cfg["workload"].split(":")[0], scheme="gpu", m=cfg["m"], n=cfg["m"], k=cfg["m"],
                nnz_a=cfg["nnz_a"], nnz_b=cfg["nnz_a"], flops=cfg["flops"], nnz_c=cfg["nnz_c"],
                max_row_size=int(det.get("max_row_size", 0)), threads=1, device=torch.cuda.get_device_name(),
                n_gpus=line["n_gpus"])
    rs = [H.BenchRecord(algorithm="kk-b200", reps=line["steps"], t_total_ms=line["ms_per_step"],
                        gflops=line["value"], roofline_frac=line["roofline"]["frac"], **base)]
    no = line.get("numeric_only") or {}
    if no.get("ms_per_step"):
        rs.append(H.BenchRecord(algorithm="kk-b200-reuse", reps=line["steps"], reuse=True,
                                t_numeric_ms=no["ms_per_step"], t_total_ms=no["ms_per_step"],
                                gflops=no.get("value") or 0.0, **base))
    H.write_bench_csv(path, rs)


def _sym_bytes(info, m, n_b):
    """SURVEY §8d symbolic-phase bytes (flops/gate pass, compress B, union)."""
    if info.compression.applied:
        return (24 * (m + 1) + 44 * info.nnz_a + 16 * (n_b + 1) + 4 * info.nnz_b + 8 * info.compressed_nnz_b
                + 8 * info.compression.compressed_flops)
    return 24 * (m + 1) + 44 * info.nnz_a + 4 * info.flops.total_flops


def _numeric_timings(args, kk, A, B, h, cols, vals, timer, barrier):
    """Numeric-only rates: the handle's default path (slot replay when
    eligible) and the hashing kernels (a handle held off the replay)."""
    os.environ["KK_NO_REPLAY"] = "1"
    h_hash = kk.symbolic(A, B)
    del os.environ["KK_NO_REPLAY"]

    def time_numeric(hh):
        for _ in range(max(args.warmup, 2)):
            kk.numeric(A, B, hh, out=(cols, vals))
        barrier()
        t = timer.run(lambda: kk.numeric(A, B, hh, out=(cols, vals)), args.steps)
        barrier()
        return t

    ms_default = time_numeric(h)
    state = h.replay_state
    ms_hash = time_numeric(h_hash) if state == 2 else ms_default
    return ms_default, ms_hash, state


def run_aa(args, kk, mats, dev, timer, barrier):
    """Configs 1, 2, 4 on one GPU: NoReuse multiply steps."""
    import torch
    a_host = mats["A"]
    A = a_host.to_device(dev)
    B = A
    h0 = kk.symbolic(A, B)
    info = h0._info()
    nnz_c = int(info.nnz_c)
    cols = torch.empty(max(nnz_c, 1), dtype=torch.int32, device=dev)
    vals = torch.empty(max(nnz_c, 1), dtype=torch.float64, device=dev)

    def step():
        h = kk.symbolic(A, B)
        kk.numeric(A, B, h, out=(cols, vals))

    for _ in range(args.warmup):
        step()
    barrier()
    l0 = kk.kernel_launch_count()
    with Clocks(dev.index) as clk:
        barrier()
        ms_total = timer.run(step, args.steps)
        barrier()
    launches = kk.kernel_launch_count() - l0
    ms_default, ms_hash, state = _numeric_timings(args, kk, A, B, h0, cols, vals, timer, barrier)
    flops = int(info.flops.total_flops)
    m = a_host.num_rows
    ms_step, ms_h = ms_total / args.steps, ms_hash / args.steps
    ms_sym = max(ms_step - ms_h, 1e-6)
    peaks, _ = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    sb = _sym_bytes(info, m, B.num_rows)
    w = 1 if info.max_row_size <= 256 else 2
    rb = 24 * (m + 1) + 28 * a_host.nnz() + (8 + w) * flops + 16 * nnz_c
    heavy = h0.heavy_path
    res = {
        "ms_total": ms_total, "flops": flops, "nnz_c": nnz_c, "m": m, "nnz_a": a_host.nnz(),
        "num_ms_total": ms_hash, "num_steps": args.steps, "launches": launches, "clocks": clk.summary(),
        "bytes_num": bytes_num(m, a_host.nnz(), flops, nnz_c),
        "num_kernel": ("numeric_slab_kernel (heavy rows, column slabs) + warp-table classes" if heavy == 2
                       else "numeric phase (hashing kernels: numeric_lp_seq/flat_kernel)"),
        "numeric_only": {"value": 2.0 * flops / (ms_default / args.steps / 1e3) / 1e9, "unit": UNIT,
                         "ms_per_step": ms_default / args.steps,
                         "path": "slot replay (kk_replay.cu)" if state == 2 else "hashing kernels",
                         "hashing_kernels": {"value": 2.0 * flops / (ms_h / 1e3) / 1e9, "unit": UNIT,
                                             "ms_per_step": ms_h}},
        "roofline_symbolic": {"bound": "hbm", "achieved": sb / (ms_sym / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                              "frac": sb / (ms_sym / 1e3) / 1e9 / hbm, "ms_per_step": ms_sym,
                              "algorithmic_bytes": sb,
                              "kernel": "symbolic phase (compress, flops, union, scan) = NoReuse step - hashing numeric",
                              "model": "24(m+1)+44nnzA+16(n+1)+4nnzB+8nnzBc+8cflops (compressed; SURVEY §8d)"},
        "roofline_replay": None if state != 2 else {
            "bound": "hbm", "achieved": rb / (ms_default / args.steps / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": rb / (ms_default / args.steps / 1e3) / 1e9 / hbm,
            "kernel": "replay_numeric_kernel (+ structure fingerprint pass)",
            "traffic": load_traffic(f"c{args.config}_replay") if args.scale == 1.0 else None,
            "algorithmic_bytes": rb, "model": "24(m+1)+28nnzA+(8+w)flops+16nnzC, w = slot bytes"},
        "detail": {"max_row_size": int(info.max_row_size), "heavy_path": heavy},
    }
    # ---- end to end through the host API (pinned host CSR in, host C out) ----
    if not args.no_e2e:
        del cols, vals, h0  # the host path allocates its own device C (c4: 116.5 GB)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        res["e2e"] = e2e_multiply_host(args, kk, a_host, nnz_c, dev, barrier, stream=timer.stream)
    return res


def e2e_multiply_host(args, kk, a_host, nnz_c, dev, barrier, stream, a_rows=None):
    import torch

    from paper_1801_03065_b200 import host
    m = a_host.num_rows if a_rows is None else a_rows[1] - a_rows[0]
    need = (m + 1) * 8 + nnz_c * 12 + a_host.nnz() * 12
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = None
    if avail is not None and need > 0.35 * avail:
        return {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                "unavailable": f"C plus inputs ({need / 1e9:.1f} GB) exceed 35% of this host's available "
                               f"memory ({avail / 1e9:.1f} GB) for pinned buffers"}
    pa = host.PinnedCsr.from_csr(a_host)
    outbuf = (torch.empty(m + 1, dtype=torch.int64).pin_memory(),
              torch.empty(max(nnz_c, 1), dtype=torch.int32).pin_memory(),
              torch.empty(max(nnz_c, 1), dtype=torch.float64).pin_memory())

    def e2e_step():
        return host.multiply_host(None if a_rows else pa, pa if a_rows else None, a_rows=a_rows, out=outbuf)

    r = e2e_step()
    assert r.c.nnz() == nnz_c
    barrier()
    ksteps = max(1, min(args.steps, 5))
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(ksteps):
        r = e2e_step()
    t1.record(stream)
    barrier()
    return {"ms_per_step": t0.elapsed_time(t1) / ksteps, "unit": UNIT, "h2d_bytes_per_step": int(r.h2d_bytes),
            "d2h_bytes_per_step": int(r.d2h_bytes), "row_blocks": r.blocks,
            "path": "host.multiply_host (C ABI): pinned host CSR in, pinned host C out, copy/compute overlap"}


def run_c3(args, kk, mats, dev, timer, barrier):
    """R*(A*P): two chained products per step, AP fed back on the device."""
    import torch
    a, p = mats["A"], mats["P"]
    A, P = a.to_device(dev), p.to_device(dev)
    R = kk.transpose(P)  # device transpose (spg_transpose), outside the timed region
    res1 = kk.multiply(A, P)
    res2 = kk.multiply(R, res1.c)
    i1, i2 = res1.handle._info(), res2.handle._info()
    fl1, fl2 = int(i1.flops.total_flops), int(i2.flops.total_flops)
    n1, n2 = int(i1.nnz_c), int(i2.nnz_c)

    def step():
        ap = kk.multiply(A, P).c
        kk.multiply(R, ap)

    for _ in range(args.warmup):
        step()
    barrier()
    l0 = kk.kernel_launch_count()
    with Clocks(dev.index) as clk:
        barrier()
        ms_total = timer.run(step, args.steps)
        barrier()
    launches = kk.kernel_launch_count() - l0
    h1, h2 = res1.handle, res2.handle
    ap_cols, ap_vals = res1.c.col_indices, res1.c.values
    rap_cols = torch.empty(max(n2, 1), dtype=torch.int32, device=dev)
    rap_vals = torch.empty(max(n2, 1), dtype=torch.float64, device=dev)
    ap = res1.c

    def reuse():
        kk.numeric(A, P, h1, out=(ap_cols, ap_vals))
        kk.numeric(R, ap, h2, out=(rap_cols, rap_vals))

    for _ in range(3):
        reuse()
    barrier()
    ms_num = timer.run(reuse, args.steps)
    barrier()
    flops = fl1 + fl2
    r_host = R.to_host()
    res = {
        "ms_total": ms_total, "flops": flops, "nnz_c": n1 + n2, "m": a.num_rows + r_host.num_rows,
        "nnz_a": a.nnz() + r_host.nnz(), "num_ms_total": ms_num, "num_steps": args.steps, "launches": launches,
        "clocks": clk.summary(),
        "bytes_num": bytes_num(a.num_rows, a.nnz(), fl1, n1) + bytes_num(r_host.num_rows, r_host.nnz(), fl2, n2),
        "num_kernel": "numeric phase of A*P and R*(AP) (hashing kernels)",
        "numeric_only": {"value": 2.0 * flops / (ms_num / args.steps / 1e3) / 1e9, "unit": UNIT,
                         "ms_per_step": ms_num / args.steps, "path": "numeric(A,P) + numeric(R,AP), structure reuse"},
        "detail": {"flops_AP": fl1, "flops_RAP": fl2, "nnz_AP": n1, "nnz_RAP": n2},
    }
    if not args.no_e2e:
        from paper_1801_03065_b200 import host
        pa, pp, pr = (host.PinnedCsr.from_csr(x) for x in (a, p, r_host))

        def e2e_step():
            r1 = host.multiply_host(pa, pp)
            o_ro, o_ci, o_v = r1._keep
            ap_h = host.PinnedCsr(a.num_rows, p.num_cols, o_ro[:a.num_rows + 1], o_ci[:n1], o_v[:n1], False)
            r2 = host.multiply_host(pr, ap_h)
            return r1, r2

        # warm-up like the device steps: the first calls fill torch's pinned
        # host cache (a call's C stays referenced until the next one returns,
        # so the cache reaches steady state on the third call)
        for _ in range(max(3, args.warmup)):
            r1, r2 = e2e_step()
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ksteps = max(1, min(args.steps, 5))
        t0.record(timer.stream)
        for _ in range(ksteps):
            r1, r2 = e2e_step()
        t1.record(timer.stream)
        barrier()
        res["e2e"] = {"ms_per_step": t0.elapsed_time(t1) / ksteps, "unit": UNIT,
                      "h2d_bytes_per_step": int(r1.h2d_bytes + r2.h2d_bytes),
                      "d2h_bytes_per_step": int(r1.d2h_bytes + r2.d2h_bytes),
                      "path": "host.multiply_host twice: A*P to pinned host AP, then R*AP (the reference's "
                              "triple product, cli.cpp:179-186, through host CSR)"}
    return res


def run_c5(args, kk, mats, dev, timer, barrier):
    """Structure reuse: one symbolic, then numeric passes with perturbed values."""
    import torch
    a = mats["A"]
    A = a.to_device(dev)
    g = torch.Generator(device=dev).manual_seed(1801)
    variants = [A.values * (1 + 1e-3 * (2 * torch.rand(A.values.shape, generator=g, device=dev,
                                                        dtype=torch.float64) - 1)) for _ in range(4)]
    As = [kk.DeviceCsr(A.num_rows, A.num_cols, A.row_offsets, A.col_indices, v, True, a.nnz()) for v in variants]
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kk.symbolic(A, A)
    t0.record()
    h = kk.symbolic(A, A)
    t1.record()
    barrier()
    ms_sym = t0.elapsed_time(t1)
    info = h._info()
    flops, nnz_c = int(info.flops.total_flops), int(info.nnz_c)
    cols = torch.empty(nnz_c, dtype=torch.int32, device=dev)
    vals = torch.empty(nnz_c, dtype=torch.float64, device=dev)
    it = [0]

    def one_pass():
        Ap = As[it[0] % 4]
        it[0] += 1
        kk.numeric(Ap, Ap, h, out=(cols, vals))

    for _ in range(max(args.warmup, 3)):
        one_pass()
    barrier()
    l0 = kk.kernel_launch_count()
    with Clocks(dev.index) as clk:
        barrier()
        ms_total = timer.run(one_pass, args.steps)
        barrier()
    launches = kk.kernel_launch_count() - l0
    ms_pass = ms_total / args.steps
    m = a.num_rows
    peaks, _ = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    w = 1 if info.max_row_size <= 256 else 2
    rb = 24 * (m + 1) + 28 * a.nnz() + (8 + w) * flops + 16 * nnz_c
    res = {
        "ms_total": ms_total, "flops": flops, "nnz_c": nnz_c, "m": m, "nnz_a": a.nnz(),
        "num_ms_total": ms_total, "num_steps": args.steps, "launches": launches, "clocks": clk.summary(),
        "bytes_num": bytes_num(m, a.nnz(), flops, nnz_c),
        "num_kernel": "numeric pass under structure reuse (%s)" % (
            "replay_numeric_kernel" if h.replay_state == 2 else "hashing kernels"),
        "numeric_only": {"value": 2.0 * flops / (ms_pass / 1e3) / 1e9, "unit": UNIT, "ms_per_step": ms_pass,
                         "path": "slot replay (kk_replay.cu)" if h.replay_state == 2 else "hashing kernels",
                         "symbolic_ms": ms_sym,
                         "amortized_1_symbolic_100_passes": {
                             "value": 100 * 2.0 * flops / ((ms_sym + 100 * ms_pass) / 1e3) / 1e9, "unit": UNIT}},
        "roofline_replay": None if h.replay_state != 2 else {
            "bound": "hbm", "achieved": rb / (ms_pass / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": rb / (ms_pass / 1e3) / 1e9 / hbm, "kernel": "replay_numeric_kernel (+ fingerprint pass)",
            "algorithmic_bytes": rb, "model": "24(m+1)+28nnzA+(8+w)flops+16nnzC, w = slot bytes"},
    }
    if not args.no_e2e:
        # per pass: the new values go up, C (row offsets, columns, values) comes
        # back — the reference's numeric returns a fresh CsrMatrix each pass
        hv = [v.cpu().pin_memory() for v in variants]
        o_ro = torch.empty(m + 1, dtype=torch.int64).pin_memory()
        o_ci = torch.empty(nnz_c, dtype=torch.int32).pin_memory()
        o_v = torch.empty(nnz_c, dtype=torch.float64).pin_memory()
        dv = torch.empty_like(variants[0])
        Ad = kk.DeviceCsr(A.num_rows, A.num_cols, A.row_offsets, A.col_indices, dv, True, a.nnz())
        ro_d = h.device_row_offsets()

        def e2e_pass(k):
            dv.copy_(hv[k % 4], non_blocking=True)
            kk.numeric(Ad, Ad, h, out=(cols, vals))
            o_ro.copy_(ro_d, non_blocking=True)
            o_ci.copy_(cols, non_blocking=True)
            o_v.copy_(vals, non_blocking=True)

        for k in range(2):
            e2e_pass(k)
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ksteps = max(1, min(args.steps, 5))
        t0.record(timer.stream)
        for k in range(ksteps):
            e2e_pass(k)
        t1.record(timer.stream)
        barrier()
        res["e2e"] = {"ms_per_step": t0.elapsed_time(t1) / ksteps, "unit": UNIT,
                      "h2d_bytes_per_step": a.nnz() * 8, "d2h_bytes_per_step": (m + 1) * 8 + nnz_c * 12,
                      "path": "numeric pass from pinned host values to pinned host C (kk.numeric, C ABI)"}
    return res


def run_sharded(args, kk, shard, mats, dev, timer, barrier, rank, world, dist):
    """Configs 1, 2, 4 on N GPUs: flop-balanced row blocks of C = A*A through
    shard.sharded_multiply (nnz all-gather and C block offsets in the step);
    B resident, then B shipped per step (broadcast / band exchange)."""
    import torch
    a_host = mats["A"]
    A = a_host.to_device(dev)
    cuts = shard.flop_cut_points(torch.cumsum(kk.row_flops(A, A), 0), world)
    lo, hi = cuts[rank], cuts[rank + 1]

    def step():
        return shard.sharded_multiply(A, A, rank, world, cuts=cuts)

    for _ in range(args.warmup):
        sh = step()
    barrier()
    l0 = kk.kernel_launch_count()
    with Clocks(dev.index) as clk:
        barrier()
        ms_total = timer.run(step, args.steps)
        barrier()
    launches = kk.kernel_launch_count() - l0
    info = sh.handle._info()
    flops, nnz_c = int(info.flops.total_flops), int(info.nnz_c)
    h = sh.handle
    cols, vals = sh.c.col_indices, sh.c.values
    blk = A.row_block(lo, hi)
    for _ in range(3):
        kk.numeric(blk, A, h, out=(cols, vals))
    barrier()
    ms_num = timer.run(lambda: kk.numeric(blk, A, h, out=(cols, vals)), args.steps)
    barrier()

    # ---- B shipped per step ----
    full = kk.DeviceCsr(A.num_rows, A.num_cols, A.row_offsets, A.col_indices, A.values, True, a_host.nnz())
    recv = kk.DeviceCsr(A.num_rows, A.num_cols, A.row_offsets.clone(), A.col_indices.clone(), A.values.clone(),
                        True, a_host.nnz())

    def step_bcast():
        b = full if rank == 0 else recv
        for t in (b.row_offsets, b.col_indices, b.values):
            dist.broadcast(t, src=0)
        shard.sharded_multiply(b, b, rank, world, cuts=cuts)

    for _ in range(2):
        step_bcast()
    barrier()
    ms_bc = timer.run(step_bcast, args.steps)
    barrier()
    bc_bytes = A.row_offsets.numel() * 8 + a_host.nnz() * 12

    # band exchange: each rank owns its rows of B (= its rows of A) and
    # receives the rows its block references from their owners (point-to-point
    # transfers: NCCL only; the gloo smoke path skips it)
    res_band = None
    if os.environ.get("KK_BENCH_BACKEND", "nccl") != "nccl":
        return _sharded_result(args, a_host, info, lo, hi, ms_total, ms_num, launches, clk, ms_bc, bc_bytes, rank,
                               None, kk, dev, barrier, timer, nnz_c, flops)
    own = shard.own_rows(A, lo, hi)
    need = shard.column_band(A, lo, hi)

    def step_band():
        band, nbytes = shard.exchange_band(own, cuts, need, rank, world, A.num_rows, A.num_cols)
        shard.sharded_multiply(band, band, rank, world, cuts=cuts)
        step_band.bytes = nbytes

    for _ in range(2):
        step_band()
    barrier()
    ms_band = timer.run(step_band, args.steps)
    barrier()
    return _sharded_result(args, a_host, info, lo, hi, ms_total, ms_num, launches, clk, ms_bc, bc_bytes, rank,
                           (ms_band, getattr(step_band, "bytes", 0)), kk, dev, barrier, timer, nnz_c, flops)


def _sharded_result(args, a_host, info, lo, hi, ms_total, ms_num, launches, clk, ms_bc, bc_bytes, rank, band, kk,
                    dev, barrier, timer, nnz_c, flops):
    m = hi - lo
    res = {
        "ms_total": ms_total, "flops": flops, "nnz_c": nnz_c, "m": m, "nnz_a": a_host.nnz(),
        "num_ms_total": ms_num, "num_steps": args.steps, "launches": launches, "clocks": clk.summary(),
        "bytes_num": bytes_num(m, int(info.nnz_a), flops, nnz_c),
        "num_kernel": "numeric phase of this rank's row block (rank 0)",
        "numeric_only": {"value": None, "unit": UNIT, "ms_per_step": ms_num / args.steps,
                         "path": "numeric on the rank's row block, B resident"},
        "with_broadcast": {"ms_total": ms_bc, "bytes": bc_bytes if rank == 0 else 0,
                           "path": "full B broadcast from rank 0 over NCCL each step, then the sharded multiply"},
    }
    if band is not None:
        res["with_band_exchange"] = {
            "ms_total": band[0], "bytes": band[1],
            "path": "each rank owns its rows of B = A and receives the rows its block references (stencil halo) "
                    "from their owners (NCCL P2P), then multiplies"}
    if not args.no_e2e:
        res["e2e"] = e2e_multiply_host(args, kk, a_host, nnz_c, dev, barrier, stream=timer.stream, a_rows=(lo, hi))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kk", choices=["kk", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--csv", default=None, help="also write the line as a BenchRecord CSV (bench.cpp:28-102)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3 if args.impl == "kk" else args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    run_gpu(args, rank, world, local)


if __name__ == "__main__":
    main()
