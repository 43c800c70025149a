"""One symbolic + four numerics (pass 2 records the slot map, 3-4 replay) on a
config, for ncu captures of replay_numeric_kernel.
Usage: python scripts/prof_replay.py cfg scale"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_03065_b200 as kk  # noqa: E402
from bench import operand_a as workload  # noqa: E402

cfg_id, scale = int(sys.argv[1]), float(sys.argv[2])
a, wl = workload(cfg_id, scale)
A = a.to_device()
h = kk.symbolic(A, A)
for p in range(4):
    st = kk.PhaseStats()
    c = kk.numeric(A, A, h, st)
    torch.cuda.synchronize()
    print(wl, "pass", p, "replay_state", h.replay_state, "numeric ms", round(st.ms, 3))
