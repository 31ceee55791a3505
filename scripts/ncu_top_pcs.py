"""Top SASS instructions by warp-stall samples with their dominant stall reasons, from an ncu report.
usage: ncu_top_pcs.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 8
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = next(r for r in rows if r and r[0] == "Address")
si = h.index("Warp Stall Sampling (All Samples)")
cols = [(i, x) for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
data = [r for r in rows if len(r) == len(h) and r[0].startswith("0x")]
tot = sum(int(r[si] or 0) for r in data)
data.sort(key=lambda r: -int(r[si] or 0))
for r in data[:n]:
    rs = sorted(((int(r[i] or 0), x[6:]) for i, x in cols if (r[i] or "0").isdigit()), reverse=True)[:3]
    print(f"{100 * int(r[si]) / tot:5.1f}%  {r[1][:58]:58s}  " + ", ".join(f"{x} {c}" for c, x in rs if c))
