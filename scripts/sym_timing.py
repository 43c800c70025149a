"""Symbolic-phase timing variants on c2 (handles kept alive vs dropped)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_03065_b200 as kk  # noqa: E402
from bench import operand_a as workload  # noqa: E402

a, _ = workload(2, 1.0)
A = a.to_device()
for _ in range(3):
    kk.symbolic(A, A)
torch.cuda.synchronize()


def timed(fn, k=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


keep = []
print("dropped", timed(lambda: kk.symbolic(A, A)))
print("kept", timed(lambda: keep.append(kk.symbolic(A, A))))
keep.clear()
h = kk.symbolic(A, A)
cols = torch.empty(h.nnz_c(), dtype=torch.int32, device="cuda")
vals = torch.empty(h.nnz_c(), dtype=torch.float64, device="cuda")
print("sym+num", timed(lambda: kk.numeric(A, A, kk.symbolic(A, A), out=(cols, vals))))
