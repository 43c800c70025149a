"""c3 triple product once (for launch lists) + host timing breakdown."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1801_03065_b200 as kk
from paper_1801_03065_b200 import generators as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
a = G.laplace3d(n); p = G.aggregation(n); r = G.transpose(p)
A, P, R = a.to_device(), p.to_device(), r.to_device()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h1 = kk.symbolic(A, P); t1 = time.perf_counter()
    c1 = kk.numeric(A, P, h1); torch.cuda.synchronize(); t2 = time.perf_counter()
    h2 = kk.symbolic(R, c1); t3 = time.perf_counter()
    c2 = kk.numeric(R, c1, h2); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"sym1 {1e3*(t1-t0):.3f} num1 {1e3*(t2-t1):.3f} sym2 {1e3*(t3-t2):.3f} num2 {1e3*(t4-t3):.3f} ms; "
          f"sym1 kernels {h1.symbolic_stats.ms:.3f} compress {h1.compress_ms:.3f}", flush=True)
