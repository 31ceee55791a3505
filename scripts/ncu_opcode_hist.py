"""Executed-instruction histogram by SASS opcode (whole kernel) from an ncu report, per tile.
usage: ncu_opcode_hist.py report.ncu-rep tiles [N]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, tiles = sys.argv[1], float(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = next(r for r in rows if r and r[0] == "Address")
ii = h.index("Instructions Executed")
ops = Counter()
for r in rows:
    if len(r) == len(h) and r[0].startswith("0x"):
        t = r[1].split()
        op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
        ops[op] += int(r[ii] or 0)
tot = sum(ops.values())
print(f"total {tot / tiles:.0f} warp instructions per tile")
for op, c in ops.most_common(n):
    print(f"{op:28s} {c / tiles:8.1f} {100 * c / tot:5.1f}%")
