"""Summarise an ncu source page (cuda,sass view): top source lines by stall samples,
with executed instructions and shared-memory / global wavefront columns."""
import csv, subprocess, sys
rep, skip = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; cur = None; res = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    def col(name):
        try:
            return int(float(r[hdr.index(name)] or 0))
        except (ValueError, IndexError):
            return 0
    if r[0] != "":
        res.append((col("Warp Stall Sampling (All Samples)"), col("Instructions Executed"),
                    col("L1 Wavefronts Shared"), col("L1 Wavefronts Shared Ideal"),
                    col("L2 Theoretical Sectors Global"), f"{cur}:{r[0]}", r[1][:80]))
ts = sum(x[0] for x in res); ti = sum(x[1] for x in res); tw = sum(x[2] for x in res)
print(f"samples {ts} warp-instructions {ti} smem-wavefronts {tw}")
print("samples   %   instrs     smem_wf  smem_ideal  l2_sect  line")
for o in sorted(res, reverse=True)[:n]:
    print(f"{o[0]:7d} {o[0]/max(ts,1)*100:5.1f} {o[1]:11d} {o[2]:11d} {o[3]:11d} {o[4]:10d} {o[5]} {o[6]}")
