"""Top SASS instructions of an ncu report's source page by stall samples and
by executed instructions.  Usage: python scripts/ncu_sass_top.py report.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = idx["Warp Stall Sampling (All Samples)"]
E = idx["Instructions Executed"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot_s = sum(float(r[S] or 0) for r in data)
tot_e = sum(float(r[E] or 0) for r in data)
print(f"total samples {tot_s:.0f}, executed warp instr {tot_e:.3e}")
agg = {}
for r in data:
    for h in stalls:
        agg[h] = agg.get(h, 0) + float(r[idx[h]] or 0)
print("stall mix:", ", ".join(f"{k[6:]} {100 * v / tot_s:.1f}%" for k, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
print("\n-- by samples --")
for k, r in sorted(enumerate(data), key=lambda t: -float(t[1][S] or 0))[:n]:
    top = sorted(((h, float(r[idx[h]] or 0)) for h in stalls), key=lambda t: -t[1])[:2]
    print(f"{k:5d} {100 * float(r[S] or 0) / tot_s:5.1f}% exe {float(r[E] or 0):.2e}  {r[1].strip()[:60]:60s} {top}")
print("\n-- by executed --")
for k, r in sorted(enumerate(data), key=lambda t: -float(t[1][E] or 0))[:n]:
    print(f"{k:5d} exe {100 * float(r[E] or 0) / tot_e:5.2f}%  {r[1].strip()[:70]}")
