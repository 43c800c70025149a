"""Per-CUDA-source-line stall samples and executed instructions of an ncu
report (captured with --import-source on).  Usage: python scripts/ncu_lines.py rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, *sys.argv[3:], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, out = None, None, []
for r in csv.reader(raw.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] and len(r) == len(hdr):
        try:
            out.append((cur, int(r[0]), r[1][:72], float(r[4] or 0), float(r[7] or 0)))
        except ValueError:
            pass
ts = sum(o[3] for o in out) or 1
te = sum(o[4] for o in out) or 1
print(f"samples {ts:.0f}, warp instructions {te:.3e}")
for key, label in ((3, "by stall samples"), (4, "by executed instructions")):
    print(f"-- {label}")
    for o in sorted(out, key=lambda o: -o[key])[:n]:
        print(f"{o[0]:16s}{o[1]:5d} {100 * o[3] / ts:5.1f}% smp {100 * o[4] / te:5.1f}% ins  {o[2]}")
