"""Per-CUDA-source-line instruction and stall-sample totals of an ncu report (compiled with
-lineinfo): where a kernel's instructions come from, by source line.

    python profiles/source_lines.py REPORT [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows, path = [], None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        path = rec[1].split("/")[-1]
        continue
    if rec[0] in ("Function Name", "Line No"):
        continue
    try:
        line = int(rec[0])
        samples, inst = int(rec[4] or 0), int(rec[7] or 0)
    except (ValueError, IndexError):
        continue
    if inst or samples:
        rows.append((inst, samples, path, line, rec[1].strip()[:90]))
tot_i = sum(r[0] for r in rows) or 1
tot_s = sum(r[1] for r in rows) or 1
print(f"# {tot_i / 1e9:.3f} G warp instructions, {tot_s} stall samples attributed to source lines")
for inst, samples, path, line, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * inst / tot_i:6.2f}% inst {100 * samples / tot_s:6.2f}% samples  {path}:{line}  {src}")
