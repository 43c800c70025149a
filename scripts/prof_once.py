"""One symbolic + one numeric on a config (for ncu captures).
Usage: python scripts/prof_once.py cfg scale [acc:scheme]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1801_03065_b200 as kk
from bench import operand_a as workload  # noqa: E402
cfg_id, scale = int(sys.argv[1]), float(sys.argv[2])
a, wl = workload(cfg_id, scale)
A = a.to_device()
cfg = kk.SpgemmConfig()
if len(sys.argv) > 3 and sys.argv[3] != "auto":
    acc, sch = (int(x) for x in sys.argv[3].split(":"))
    cfg = kk.SpgemmConfig(accumulator=acc, scheme=sch)
h = kk.symbolic(A, A, cfg)
st = kk.PhaseStats()
c = kk.numeric(A, A, h, st)
torch.cuda.synchronize()
print(wl, "nnz_c", h.nnz_c(), "numeric ms", st.ms)
