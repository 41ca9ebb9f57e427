"""Per-kernel summary of an ncu --csv launch list (gpu__time_duration.sum): python tools/launch_summary.py f.csv"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")) / 1000.0)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':70s} {'launches':>8s} {'mean_us':>9s} {'total_us':>9s} share")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} {len(v):8d} {sum(v)/len(v):9.1f} {sum(v):9.1f} {100*sum(v)/tot:5.1f}%")
