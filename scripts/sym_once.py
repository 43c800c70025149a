"""One symbolic pass (and with --numeric one hashing numeric pass) of a bench
config, as an ncu target.  Usage: python scripts/sym_once.py cfg [scale] [--numeric]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_03065_b200 as kk  # noqa: E402
from bench import operand_a  # noqa: E402

cfg = int(sys.argv[1])
scale = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 1.0
a, _ = operand_a(cfg, scale)
A = a.to_device()
h = kk.symbolic(A, A)
torch.cuda.synchronize()
print("nnz_c", h.nnz_c())
if "--numeric" in sys.argv:
    kk.numeric(A, A, h)
    torch.cuda.synchronize()
