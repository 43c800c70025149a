"""Three numeric passes on one handle (the third is the slot replay), as an ncu
target.  Usage: python scripts/replay_once.py cfg [scale]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_03065_b200 as kk  # noqa: E402
from bench import operand_a  # noqa: E402

cfg = int(sys.argv[1])
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
a, _ = operand_a(cfg, scale)
A = a.to_device()
h = kk.symbolic(A, A)
c = kk.numeric(A, A, h)
for _ in range(2):
    kk.numeric(A, A, h, out=(c.col_indices, c.values))
torch.cuda.synchronize()
print("replay state", h.replay_state)
