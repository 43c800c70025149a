"""Key ncu metrics of captured launches -> a markdown table (profiles/).
Usage: python scripts/kernel_report.py out.md label=report.ncu-rep [...]
Every launch in each report becomes a row."""
import csv
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def rows(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) < 3:
        return []
    hh, uu = rr[0], rr[1]
    out = []
    for r in rr[2:]:
        d = {hh[i]: (r[i], uu[i]) for i in range(min(len(hh), len(r)))}
        out.append(d)
    return out


def main():
    dst = sys.argv[1]
    lines = ["| label | kernel | " + " | ".join(n for _, n in WANT) + " |",
             "|---|---|" + "---|" * len(WANT)]
    for arg in sys.argv[2:]:
        label, rep = arg.split("=", 1)
        for d in rows(rep):
            name = d.get("Kernel Name", ("?", ""))[0].split("(")[0][:48]
            cells = []
            for key, _ in WANT:
                v, u = d.get(key, ("", ""))
                cells.append(f"{v} {u}".strip() if v else "-")
            lines.append(f"| {label} | `{name}` | " + " | ".join(cells) + " |")
    with open(dst, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
