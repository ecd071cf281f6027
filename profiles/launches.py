"""Summarise an ncu launch list (gpu__time_duration.sum CSV of bench.py's timed region).

    python profiles/launches.py gpurun_out/launches_TAG_WL.csv "header line"
"""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))
        if r.get("Metric Name") == "gpu__time_duration.sum"]
tot = collections.Counter()
for r in rows:
    tot[r["Kernel Name"]] += float(r["Metric Value"])
all_ns = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"# {len(rows)} launches inside the timed region; share of device time per kernel:")
for k, v in tot.most_common():
    print(f"{100 * v / all_ns:8.3f}%  {v / 1e3:14.1f} us total  {k[:90]}")
print("\n# per launch:")
for r in rows:
    print(f"{float(r['Metric Value']):14.0f} ns  {r['Kernel Name'][:90]}")
