"""Per-kernel device time of one NoReuse multiply and one numeric-only pass
(torch.profiler / CUPTI), for quick phase breakdowns between ncu captures.
Usage: python scripts/kprof.py cfg [scale] [--reps R]"""
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_03065_b200 as kk  # noqa: E402
from bench import operand_a as workload  # noqa: E402


def main():
    cfg_id = int(sys.argv[1])
    scale = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 1.0
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 1
    a, wl = workload(cfg_id, scale)
    A = a.to_device()
    h = kk.symbolic(A, A)
    c = kk.numeric(A, A, h)
    torch.cuda.synchronize()
    # wall timings
    for label, fn in (("symbolic", lambda: kk.symbolic(A, A)),
                      ("numeric", lambda: kk.numeric(A, A, h, out=(c.col_indices, c.values)))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"{label}: {e0.elapsed_time(e1) / reps:.3f} ms (events, {reps} reps)")
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        h2 = kk.symbolic(A, A)
        kk.numeric(A, A, h2, out=(c.col_indices, c.values))
        torch.cuda.synchronize()
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name.split("(")[0][:70]
            tot[name] += ev.device_time_total / 1e3 if hasattr(ev, "device_time_total") else ev.cuda_time_total / 1e3
            cnt[name] += 1
    print(wl, "flops", h.flops.total_flops, "nnz_c", h.nnz_c(), "max_row", h.max_row_size)
    for k, v in sorted(tot.items(), key=lambda t: -t[1]):
        print(f"  {v:9.3f} ms  x{cnt[k]:3d}  {k}")


if __name__ == "__main__":
    main()
