"""Per-kernel launch counts, average duration and share of an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`).  usage: launch_shares.py X.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
acc = defaultdict(list)
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        acc[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in acc.values())
print("| kernel | launches | avg us | share |\n|---|---|---|---|")
for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    print(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
