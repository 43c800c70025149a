"""Timeline of one host.multiply_host call on a config (event marks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import operand_a as workload  # noqa: E402
from paper_1801_03065_b200 import host  # noqa: E402

cfg_id, scale = int(sys.argv[1]), float(sys.argv[2])
blocks = int(sys.argv[3]) if len(sys.argv) > 3 else None
a, wl = workload(cfg_id, scale)
pa = host.PinnedCsr.from_csr(a)
r = host.multiply_host(pa, blocks=blocks)
out = (torch.empty(a.num_rows + 1, dtype=torch.int64).pin_memory(),
       torch.empty(r.c.nnz(), dtype=torch.int32).pin_memory(),
       torch.empty(r.c.nnz(), dtype=torch.float64).pin_memory())
del r
for _ in range(2):
    tl = []
    r = host.multiply_host(pa, blocks=blocks, out=out, timeline=tl)
    t0 = tl[0][1]
    print(wl, "blocks", r.blocks)
    for label, ev in tl:
        print(f"  {t0.elapsed_time(ev):9.2f} ms  {label}")
