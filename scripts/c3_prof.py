"""Kernel breakdown of one c3 step (A*P then R*(AP)) via torch.profiler.
Usage: python scripts/c3_prof.py"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_03065_b200 as kk  # noqa: E402
from paper_1801_03065_b200 import generators as G  # noqa: E402
from bench import workload  # noqa: E402

mats, wl = workload(3, 1.0, G)
A, P = mats["A"].to_device(), mats["P"].to_device()
R = kk.transpose(P)
for _ in range(3):
    kk.multiply(R, kk.multiply(A, P).c)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
ap = kk.multiply(A, P).c
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ap2 = kk.multiply(A, P).c
    torch.cuda.synchronize()
    kk.multiply(R, ap2)
    torch.cuda.synchronize()
tot, cnt = defaultdict(float), defaultdict(int)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.split("(")[0][:80]
        tot[name] += ev.device_time_total / 1e3
        cnt[name] += 1
for k, v in sorted(tot.items(), key=lambda t: -t[1]):
    print(f"  {v:9.3f} ms  x{cnt[k]:3d}  {k}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for label, fn in (("A*P multiply", lambda: kk.multiply(A, P)), ("R*AP multiply", lambda: kk.multiply(R, ap))):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / 10:.3f} ms")
