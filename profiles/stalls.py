"""Per-opcode and per-instruction stall-sample summary of an ncu report (source page)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, vals = rows[0], rows[2]
print("stall reasons (warp-cycles per issued instruction):")
for i, h in enumerate(hdr):
    if "average_warps_issue_stalled" in h and "per_issue_active" in h:
        v = float(vals[i])
        if v > 0.05:
            print(f"  {h.split('stalled_')[1].replace('_per_issue_active.ratio', ''):28s} {v:.3f}")
for k in ("smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "gpu__time_duration.sum"):
    print(f"{k:60s} {vals[hdr.index(k)]}")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
iS, iSrc, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
tot = sum(int(r[iS]) for r in data)
by, ex = collections.Counter(), collections.Counter()
for r in data:
    op = r[iSrc].strip().split()
    op = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
    by[op] += int(r[iS])
    ex[op] += int(r[iE] or 0)
print("opcode: %samples, executed (M)")
print("  " + ", ".join(f"{k} {v / tot * 100:.1f}% {ex[k] / 1e6:.0f}M" for k, v in by.most_common(top)))
order = sorted(range(len(data)), key=lambda i: -int(data[i][iS]))
print("hottest instructions:")
for i in order[:top]:
    r = data[i]
    print(f"  {int(r[iS]) / tot * 100:5.2f}% line {i:5d} exec {r[iE]:>10s}  {r[iSrc].strip()[:70]}")
