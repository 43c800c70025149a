"""Secondary bench lines for BASELINE.json configs 1, 3, 4, 5 (the driver's
bench.py runs config 2, the headline).  Same JSON schema as bench.py; one line
per config.  Usage: python scripts/bench_configs.py [1,3,4,5] [--steps K]

  c1  C=A*A, 2D 5-point 1000^2                          sym+num per step
  c3  R*(A*P): 3D 27-point 128^3, 2x2x2 aggregation P   both products per step (AP fed back
                                                         unsorted, on device)
  c4  C=A*A, R-MAT s20 ef16                             sym+num per step
  c5  1 symbolic + N numeric passes, values perturbed   value = N*2*flops / (t_sym + sum t_num)
      per pass vals*(1+1e-3*U_p), 3D 27-point 200^3

CPU baseline = the reference library (oracle/_ref) on this host's cores, full
problem where it fits the time budget, otherwise a row sample (labelled).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_03065_b200 as kk  # noqa: E402
from paper_1801_03065_b200 import generators as G  # noqa: E402


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def base_line(wl, value, ms, steps, warmup, extra):
    line = {"metric": bench.METRIC, "value": value, "unit": bench.UNIT, "n_gpus": 1, "steps": steps,
            "warmup": warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": {"workload": wl}}
    line.update(extra)
    return line


def cpu_ref(fn_mult, fl, label):
    """fn_mult() -> seconds of one reference multiply; returns cpu_baseline."""
    from oracle.oracle import reference_available
    times = [fn_mult() for _ in range(2)]
    t = float(np.mean(times))
    return {"value": 2.0 * fl / t / 1e9, "unit": bench.UNIT, "cores": os.cpu_count(),
            "kind": "reference" if reference_available() else "port", "sample": label}


def c1(steps, warmup):
    a, wl = bench.workload(1, 1.0)
    A = a.to_device()
    h = kk.symbolic(A, A)
    fl = h.flops.total_flops
    ms = timed(lambda: kk.numeric(A, A, kk.symbolic(A, A)), steps, warmup)
    cols = torch.empty(h.nnz_c(), dtype=torch.int32, device="cuda")
    vals = torch.empty(h.nnz_c(), dtype=torch.float64, device="cuda")
    msn = timed(lambda: kk.numeric(A, A, h, out=(cols, vals)), steps, warmup)
    rate, cores, kind, sample = bench.cpu_reference_rate(a)
    return base_line(wl, 2 * fl / ms / 1e6, ms, steps, warmup, {
        "numeric_only": {"value": 2 * fl / msn / 1e6, "ms_per_step": msn},
        "cpu_baseline": {"value": rate, "unit": bench.UNIT, "cores": cores, "kind": kind, "sample": sample}})


def c3(steps, warmup):
    n = 128
    a = G.laplace3d(n)
    p = G.aggregation(n)
    A, P = a.to_device(), p.to_device()
    R = kk.transpose(P)  # device transpose (spg_transpose), outside the timed region
    r = R.to_host()      # the CPU baseline's R
    res1 = kk.multiply(A, P)
    res2 = kk.multiply(R, res1.c)
    fl1, fl2 = res1.handle.flops.total_flops, res2.handle.flops.total_flops

    def step():
        ap = kk.multiply(A, P).c
        kk.multiply(R, ap)

    ms = timed(step, steps, warmup)

    # numeric-only reuse of the chain (A's values change, structure fixed):
    # two numeric passes per step, plain and captured in one CUDA graph
    h1, h2 = res1.handle, res2.handle
    ap_cols, ap_vals = res1.c.col_indices, res1.c.values
    rap_cols = torch.empty(max(h2.nnz_c(), 1), dtype=torch.int32, device="cuda")
    rap_vals = torch.empty(max(h2.nnz_c(), 1), dtype=torch.float64, device="cuda")
    ap = res1.c

    def reuse():
        kk.numeric(A, P, h1, out=(ap_cols, ap_vals))
        kk.numeric(R, ap, h2, out=(rap_cols, rap_vals))

    ms_reuse = timed(reuse, max(steps, 20), warmup)
    s_cap = torch.cuda.Stream()
    s_cap.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s_cap):
        for _ in range(2):
            kk.numeric(A, P, h1, stream=s_cap, out=(ap_cols, ap_vals))
            kk.numeric(R, ap, h2, stream=s_cap, out=(rap_cols, rap_vals))
        with torch.cuda.graph(g, stream=s_cap):
            kk.numeric(A, P, h1, stream=s_cap, out=(ap_cols, ap_vals))
            kk.numeric(R, ap, h2, stream=s_cap, out=(rap_cols, rap_vals))
    torch.cuda.current_stream().wait_stream(s_cap)
    ms_graph = timed(g.replay, max(steps, 20), warmup)

    from oracle.oracle import Reference, reference_available
    cpu = None
    if reference_available():
        ref = Reference()
        ap_ro = res1.handle.c_row_offsets
        apc = res1.c.to_host()

        def one():
            ms1, _ = ref.multiply_ms(a, p, worker_count=os.cpu_count())
            ms2, _ = ref.multiply_ms(r, apc, worker_count=os.cpu_count())
            return (ms1 + ms2) / 1e3
        cpu = cpu_ref(one, fl1 + fl2, "full c3: reference multiply(A,P) + multiply(R,AP), mean of 2")
        del ap_ro
    return base_line(f"c3: R*(A*P), 3D 27-point {n}^3, 2x2x2 aggregation P, R=P^T, fp64", 2 * (fl1 + fl2) / ms / 1e6,
                     ms, steps, warmup, {"config_detail": {"flops_AP": fl1, "flops_RAP": fl2,
                                                           "nnz_AP": res1.handle.nnz_c(),
                                                           "nnz_RAP": res2.handle.nnz_c()},
                                         "numeric_only": {"value": 2 * (fl1 + fl2) / ms_reuse / 1e6,
                                                          "ms_per_step": ms_reuse},
                                         "numeric_only_cuda_graph": {"value": 2 * (fl1 + fl2) / ms_graph / 1e6,
                                                                     "ms_per_step": ms_graph},
                                         "cpu_baseline": cpu})


def c4(steps, warmup):
    a, wl = bench.workload(4, 1.0)
    A = a.to_device()
    cfg = kk.SpgemmConfig(pool_budget_bytes=16 << 30)
    h = kk.symbolic(A, A, cfg)
    fl = h.flops.total_flops
    nnz = h.nnz_c()
    cols = torch.empty(nnz, dtype=torch.int32, device="cuda")
    vals = torch.empty(nnz, dtype=torch.float64, device="cuda")

    def step():
        hh = kk.symbolic(A, A, cfg)
        kk.numeric(A, A, hh, out=(cols, vals))

    ms = timed(step, steps, warmup)
    msn = timed(lambda: kk.numeric(A, A, h, out=(cols, vals)), steps, warmup)
    from oracle.oracle import Oracle, Reference, reference_available
    cpu = None
    if reference_available():
        ref = Reference()
        s = bench.row_sample(a, 64)
        _, fls, _ = Oracle().flops_stats(s, a)
        cpu = cpu_ref(lambda: ref.multiply_ms(s, a, worker_count=os.cpu_count())[0] / 1e3, fls,
                      "rows 0::64 of A x full B (full C = 116.5 GB exceeds host RAM); rate extrapolated by "
                      "sampled flops")
    return base_line(wl, 2 * fl / ms / 1e6, ms, steps, warmup, {
        "numeric_only": {"value": 2 * fl / msn / 1e6, "ms_per_step": msn},
        "config_detail": {"flops": fl, "nnz_c": nnz, "max_row_size": h.max_row_size, "pool_budget_gib": 16},
        "cpu_baseline": cpu})


def c5(passes, warmup):
    a, wl = bench.workload(5, 1.0)
    A = a.to_device()
    g = torch.Generator(device="cuda").manual_seed(1801)
    variants = [A.values * (1 + 1e-3 * (2 * torch.rand(A.values.shape, generator=g, device="cuda",
                                                        dtype=torch.float64) - 1)) for _ in range(4)]
    As = [kk.DeviceCsr(A.num_rows, A.num_cols, A.row_offsets, A.col_indices, v, True, a.nnz()) for v in variants]
    torch.cuda.synchronize()
    ms_sym = timed(lambda: kk.symbolic(A, A), 1, 1)
    h = kk.symbolic(A, A)
    fl = h.flops.total_flops
    cols = torch.empty(h.nnz_c(), dtype=torch.int32, device="cuda")
    vals = torch.empty(h.nnz_c(), dtype=torch.float64, device="cuda")
    it = [0]

    def one_pass():
        Ap = As[it[0] % 4]
        it[0] += 1
        kk.numeric(Ap, Ap, h, out=(cols, vals))

    ms_num = timed(one_pass, passes, warmup)
    total_ms = ms_sym + passes * ms_num
    from oracle.oracle import Oracle, Reference, reference_available
    cpu = None
    if reference_available():
        ref = Reference()
        s = bench.row_sample(a, 64)
        _, fls, _ = Oracle().flops_stats(s, a)
        rh = ref.symbolic(s, a, worker_count=os.cpu_count())
        rh.set_workers(os.cpu_count())

        def one():
            t0 = time.perf_counter()
            rh.numeric()
            return time.perf_counter() - t0
        cpu = cpu_ref(one, fls, "numeric-only pass of the reference on rows 0::64 of A x full B, mean of 2")
    return base_line(wl + f", 1 symbolic + {passes} numeric passes (perturbed values)",
                     passes * 2 * fl / total_ms / 1e6, total_ms / passes, passes, warmup, {
                         "numeric_only": {"value": 2 * fl / ms_num / 1e6, "ms_per_step": ms_num},
                         "symbolic_ms": ms_sym, "cpu_baseline": cpu})


if __name__ == "__main__":
    which = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-")
                              else "1,3,4,5").split(",")]
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 5
    for c in which:
        fn = {1: c1, 3: c3, 4: c4, 5: c5}[c]
        line = fn(100 if c == 5 else steps, 3 if c != 4 else 1)
        print(json.dumps(line), flush=True)
