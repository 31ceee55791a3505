"""Stall reasons summed over SASS instructions between the first and last instruction matching a
pattern (e.g. MUFU.EX2) of an ncu report.  usage: ncu_sass_region.py report PATTERN"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep, pat = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = next(r for r in rows if r and r[0] == "Address")
body = [r for r in rows if len(r) == len(h) and r[0].startswith("0x")]
idx = [i for i, r in enumerate(body) if re.search(pat, r[1])]
lo, hi = idx[0], idx[-1]
cols = [(i, n) for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
tot = Counter()
samples = inst = 0
ops = Counter()
for r in body[lo:hi + 1]:
    samples += int(r[si] or 0)
    inst += int(r[ii] or 0)
    ops[r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]] += int(r[ii] or 0)
    for i, n in cols:
        tot[n] += int(r[i] or 0)
allsamp = sum(int(r[si] or 0) for r in body)
print(f"region {lo}..{hi} ({hi - lo + 1} SASS lines): {samples} of {allsamp} samples, {inst} warp instr")
print("stalls:", ", ".join(f"{k[6:]}={v}" for k, v in tot.most_common(8)))
print("ops:", ", ".join(f"{k}={v}" for k, v in ops.most_common(14)))
