"""Per-CUDA-source-line executed instructions and stall samples of an ncu report.

    python profiles/lines.py REPORT [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = []
fname = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No",) or r[0] == "":
        continue
    try:
        agg.append((fname, int(r[0]), r[1].strip()[:70], int(r[4] or 0), int(r[7] or 0)))
    except ValueError:
        pass
tot_s = sum(a[3] for a in agg) or 1
tot_e = sum(a[4] for a in agg) or 1
print(f"total executed warp instructions {tot_e / 1e9:.2f} G, samples {tot_s}")
for f, ln, src, smp, ex in sorted(agg, key=lambda a: -a[4])[:top]:
    print(f"{ex / tot_e * 100:5.1f}% inst {smp / tot_s * 100:5.1f}% smp  {f}:{ln:<4d} {src}")
