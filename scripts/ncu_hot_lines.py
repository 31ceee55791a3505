"""Top CUDA source lines by warp-stall samples from an ncu report (source page, cuda+sass view).
usage: ncu_hot_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
lines = [r for r in rows if len(r) > si and r[0].isdigit() and r[2] == "-"]
tot = sum(int(r[si] or 0) for r in lines)
print(f"total samples {tot}")
for r in sorted(lines, key=lambda r: -int(r[si] or 0))[:n]:
    s = int(r[si] or 0)
    print(f"{r[0]:>5} {100 * s / tot:5.1f}% inst {r[ii]:>10} | {r[1][:110]}")
