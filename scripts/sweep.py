"""Variant sweep on one config: time symbolic and numeric for each forced
(accumulator, scheme) with CUDA events.  Usage: python scripts/sweep.py [cfg] [scale]"""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
os.environ.setdefault("KK_NO_REPLAY", "1")  # time the hashing kernels (bench.py times the replay)
import paper_1801_03065_b200 as kk
from bench import operand_a as workload

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["auto", "1:0", "1:1", "2:0", "2:1"]
a, wl = workload(cfg_id, scale)
A = a.to_device()
print(wl, flush=True)

def timeit(fn, reps=int(os.environ.get("SWEEP_REPS", "3"))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for v in variants:
    if v.startswith("auto"):
        cfg = kk.SpgemmConfig()
        if "@" in v:
            cfg.lp_max_occupancy = float(v.split("@")[1])
    else:
        acc, sch = (int(x) for x in v.split(":"))
        cfg = kk.SpgemmConfig(accumulator=acc, scheme=sch)
    h = kk.symbolic(A, A, cfg)
    info = h._info()
    nnz = info.nnz_c
    cols = torch.empty(nnz, dtype=torch.int32, device="cuda")
    vals = torch.empty(nnz, dtype=torch.float64, device="cuda")
    t_sym = timeit(lambda: kk.symbolic(A, A, cfg))
    t_num = timeit(lambda: kk.numeric(A, A, h, out=(cols, vals)))
    fl = info.flops.total_flops
    print(json.dumps({"variant": v, "sym_ms": round(t_sym, 3), "num_ms": round(t_num, 3),
                      "symnum_gflops": round(2 * fl / (t_sym + t_num) / 1e6, 1),
                      "num_gflops": round(2 * fl / t_num / 1e6, 1),
                      "compress_ms": round(info.compress_ms, 3), "sym_kernel_ms": round(info.symbolic_stats.ms, 3),
                      "sym_choice": [info.symbolic_choice.accumulator, info.symbolic_choice.scheme],
                      "num_choice": [info.numeric_choice.accumulator, info.numeric_choice.scheme]}), flush=True)
