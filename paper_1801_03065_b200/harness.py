"""Benchmark/CSV harness — the reference's `bench` and
`profile` reporting, driven by the GPU engine.

* ``BenchRecord`` / ``write_bench_csv`` / ``read_bench_csv``: the reference's
  22-column results schema byte for byte (bench.hpp:14-36, bench.cpp:28-102),
  so GPU rows and rows produced by the reference CLI can be profiled together;
  GPU-only columns (device, n_gpus, roofline fraction) go to a sidecar
  ``<out>.gpu.csv``.
* ``bench_problem``: warmup + ``reps`` timed full multiplies, optionally
  ``reuse`` numeric-only repetitions against one handle (cli.cpp:132-174), timed
  with CUDA events on device-resident operands.
* ``compute_profile`` / ``write_profile_csv``: the Dolan-Moré performance
  profile (bench.cpp:104-175).

    python -m paper_1801_03065_b200.harness bench --config 2 --reps 5 --reuse 5 --out r.csv
    python -m paper_1801_03065_b200.harness profile --in r.csv --out p.csv --points 50
"""
from __future__ import annotations

import argparse
import csv
import dataclasses
import math
import os
import sys
from typing import Dict, List

HEADER = ("problem,algorithm,scheme,m,n,k,nnz_a,nnz_b,flops,max_row_flops,nnz_c,"
          "max_row_size,cf,cmrf,threads,reps,reuse,t_compress_ms,t_symbolic_ms,"
          "t_numeric_ms,t_total_ms,gflops")


@dataclasses.dataclass
class BenchRecord:
    problem: str = ""
    algorithm: str = ""
    scheme: str = ""
    m: int = 0
    n: int = 0
    k: int = 0
    nnz_a: int = 0
    nnz_b: int = 0
    flops: int = 0
    max_row_flops: int = 0
    nnz_c: int = 0
    max_row_size: int = 0
    cf: float = 1.0
    cmrf: float = 1.0
    threads: int = 1
    reps: int = 0
    reuse: bool = False
    t_compress_ms: float = 0.0
    t_symbolic_ms: float = 0.0
    t_numeric_ms: float = 0.0
    t_total_ms: float = 0.0
    gflops: float = 0.0
    # GPU sidecar columns
    device: str = ""
    n_gpus: int = 1
    roofline_frac: float = 0.0


def _row(r: BenchRecord) -> str:
    # bench.cpp:42-52 printf format
    return (f"{r.problem},{r.algorithm},{r.scheme},{r.m},{r.n},{r.k},{r.nnz_a},{r.nnz_b},{r.flops},"
            f"{r.max_row_flops},{r.nnz_c},{r.max_row_size},{r.cf:.6f},{r.cmrf:.6f},{r.threads},{r.reps},"
            f"{1 if r.reuse else 0},{r.t_compress_ms:.6f},{r.t_symbolic_ms:.6f},{r.t_numeric_ms:.6f},"
            f"{r.t_total_ms:.6f},{r.gflops:.6f}")


def write_bench_csv(path: str, records: List[BenchRecord]) -> None:
    with open(path, "w") as f:
        f.write(HEADER + "\n")
        for r in records:
            f.write(_row(r) + "\n")
    with open(os.path.splitext(path)[0] + ".gpu.csv", "w") as f:
        f.write("problem,algorithm,reuse,device,n_gpus,roofline_frac\n")
        for r in records:
            f.write(f"{r.problem},{r.algorithm},{1 if r.reuse else 0},{r.device},{r.n_gpus},{r.roofline_frac:.6f}\n")


def read_bench_csv(path: str) -> List[BenchRecord]:
    """bench.cpp:55-102: exact header, field count and types checked."""
    with open(path) as f:
        lines = f.read().splitlines()
    if not lines:
        raise ValueError("empty results file (line 1)")
    if lines[0].split(",") != HEADER.split(","):
        raise ValueError("unexpected results header (line 1)")
    out = []
    for lineno, line in enumerate(lines[1:], start=2):
        if not line:
            continue
        f = line.split(",")
        if len(f) != 22:
            raise ValueError(f"wrong field count (line {lineno})")
        try:
            out.append(BenchRecord(f[0], f[1], f[2], int(f[3]), int(f[4]), int(f[5]), int(f[6]), int(f[7]),
                                   int(f[8]), int(f[9]), int(f[10]), int(f[11]), float(f[12]), float(f[13]),
                                   int(f[14]), int(f[15]), int(f[16]) != 0, float(f[17]), float(f[18]),
                                   float(f[19]), float(f[20]), float(f[21])))
        except ValueError:
            raise ValueError(f"malformed field (line {lineno})") from None
    return out


@dataclasses.dataclass
class PerformanceProfile:
    x: List[float]
    methods: List[str]
    counts: List[List[int]]


def compute_profile(records: List[BenchRecord], grid_points: int = 50) -> PerformanceProfile:
    """Dolan-Moré profile (bench.cpp:104-156): for each method and slowdown
    factor x on a log grid from 1 to the largest ratio, the number of problems
    solved within x of the per-problem best time."""
    if grid_points < 1:
        raise ValueError("compute_profile: grid_points must be >= 1")
    best: Dict[str, float] = {}
    times: Dict[str, Dict[str, float]] = {}
    for r in records:
        if r.t_total_ms <= 0.0:
            continue
        per = times.setdefault(r.algorithm, {})
        per[r.problem] = r.t_total_ms if r.problem not in per else min(per[r.problem], r.t_total_ms)
        if r.problem not in best or r.t_total_ms < best[r.problem]:
            best[r.problem] = r.t_total_ms
    if len(times) < 2:
        raise ValueError("compute_profile: need at least two methods")
    max_ratio = 1.0
    for per in times.values():
        for prob, t in per.items():
            max_ratio = max(max_ratio, t / best[prob])
    if max_ratio == 1.0 or grid_points == 1:
        xs = [1.0]
    else:
        xs = [math.pow(max_ratio, g / (grid_points - 1)) for g in range(grid_points)]
    methods = sorted(times)  # std::map iteration order
    counts = [[sum(1 for prob, t in times[m].items() if t / best[prob] <= x) for x in xs] for m in methods]
    return PerformanceProfile(xs, methods, counts)


def write_profile_csv(path: str, p: PerformanceProfile) -> None:
    with open(path, "w") as f:
        f.write("x" + "".join("," + m for m in p.methods) + "\n")
        for g, x in enumerate(p.x):
            f.write(f"{x:.9g}" + "".join(f",{p.counts[m][g]}" for m in range(len(p.methods))) + "\n")


def bench_problem(problem: str, a, b, cfg=None, reps: int = 5, reuse: int = 0, label: str = "auto",
                  scheme: str = "seq") -> List[BenchRecord]:
    """cli.cpp:132-174 on the GPU: warmup + `reps` timed multiplies (CUDA
    events), optional reuse record of numeric-only passes."""
    import torch
    import paper_1801_03065_b200 as kk
    from bench import bytes_num as algorithmic_bytes_numeric, _peaks
    da, db = kk._dev(a), kk._dev(b)
    warm = kk.multiply(da, db, cfg)
    h = warm.handle
    base = dict(problem=problem, scheme=scheme, m=h.m, n=h.n, k=h.k, nnz_a=h.nnz_a, nnz_b=h.nnz_b,
                nnz_c=h.nnz_c(), flops=h.flops.total_flops, max_row_flops=h.flops.max_row_flops,
                max_row_size=h.max_row_size, cf=h.compression.cf, cmrf=h.compression.cmrf, threads=1,
                device=torch.cuda.get_device_name(), n_gpus=1)
    rec = BenchRecord(algorithm=label, reps=reps, **base)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        e0.record()
        res = kk.multiply(da, db, cfg)
        e1.record()
        torch.cuda.synchronize()
        rec.t_total_ms += e0.elapsed_time(e1)
        rec.t_compress_ms += res.handle.compress_ms
        rec.t_symbolic_ms += res.handle.symbolic_stats.ms
        rec.t_numeric_ms += res.numeric_stats.ms
    for f in ("t_total_ms", "t_compress_ms", "t_symbolic_ms", "t_numeric_ms"):
        setattr(rec, f, getattr(rec, f) / max(reps, 1))
    rec.gflops = 2.0 * rec.flops / (rec.t_total_ms * 1e6) if rec.t_total_ms > 0 else 0.0
    hbm = float(_peaks()[0].get("hbm_gbs", 6650.0))
    nbytes = algorithmic_bytes_numeric(h.m, h.nnz_a, h.flops.total_flops, h.nnz_c())
    rec.roofline_frac = nbytes / (rec.t_numeric_ms * 1e6) / hbm if rec.t_numeric_ms > 0 else 0.0
    out = [rec]
    if reuse > 0:
        ru = BenchRecord(algorithm=label + "-reuse", reps=reuse, reuse=True, **base)
        kk.numeric(da, db, h)
        for _ in range(reuse):
            st = kk.PhaseStats()
            kk.numeric(da, db, h, st)
            ru.t_numeric_ms += st.ms
        ru.t_numeric_ms /= reuse
        ru.t_total_ms = ru.t_numeric_ms
        ru.gflops = 2.0 * ru.flops / (ru.t_total_ms * 1e6) if ru.t_total_ms > 0 else 0.0
        ru.roofline_frac = nbytes / (ru.t_numeric_ms * 1e6) / hbm if ru.t_numeric_ms > 0 else 0.0
        out.append(ru)
    return out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="harness")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench")
    b.add_argument("--config", type=int, default=2)
    b.add_argument("--scale", type=float, default=1.0)
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--reuse", type=int, default=0)
    b.add_argument("--out", required=True)
    p = sub.add_parser("profile")
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--points", type=int, default=50)
    args = ap.parse_args(argv)
    if args.cmd == "profile":
        write_profile_csv(args.out, compute_profile(read_bench_csv(args.inp), args.points))
        return 0
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from bench import operand_a
    a, wl = operand_a(args.config, args.scale)
    recs = bench_problem(f"c{args.config}", a, a, reps=args.reps, reuse=args.reuse)
    write_bench_csv(args.out, recs)
    print(f"wrote {len(recs)} record(s) for {wl} to {args.out}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
