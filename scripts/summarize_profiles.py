"""Summarise ncu outputs into profiles/ (tracked):
  launches CSV (gpu__time_duration.sum per launch) -> per-kernel totals and shares
  full capture (.ncu-rep) -> key metrics incl. dram bytes -> profiles/traffic.json
Usage: python scripts/summarize_profiles.py <tag> <launches.csv> <full.ncu-rep> <traffic-key>"""
import csv, json, os, subprocess, sys
from collections import defaultdict
tag, launches, rep, key = sys.argv[1:5]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = []
rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi and r[vi]:
        agg[r[ki].split("(")[0][:60]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
out.append(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
out.append("| kernel | launches | total ms | avg us | share |\n|---|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    out.append(f"| `{k}` | {len(v)} | {sum(v)/1e6:.3f} | {sum(v)/len(v)/1e3:.1f} | {sum(v)/tot*100:.1f}% |")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hh, uu = rr[0], rr[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
out.append(f"\n## full capture ({os.path.basename(rep)}; ncu --set full, one launch)\n")
out.append("| metric | value | unit |\n|---|---|---|")
traffic = None
for r in rr[2:]:
    d = {hh[i]: (r[i], uu[i]) for i in range(len(hh))}
    for w in want:
        if w in d:
            out.append(f"| {w} | {d[w][0]} | {d[w][1]} |")
    def to_bytes(v, u):
        v = float(v.replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    traffic = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
    break
os.makedirs(os.path.join(root, "profiles"), exist_ok=True)
with open(os.path.join(root, "profiles", f"{tag}.md"), "w") as f:
    f.write("\n".join(out) + "\n")
tp = os.path.join(root, "profiles", "traffic.json")
tj = json.load(open(tp)) if os.path.exists(tp) else {}
tj[key] = traffic
json.dump(tj, open(tp, "w"), indent=1)
print("\n".join(out))
