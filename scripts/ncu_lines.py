"""Summarise an `ncu --page source --csv --print-source cuda,sass` export: per CUDA source line,
samples, instructions and the dominant stall reasons.  usage: ncu_lines.py file.csv [lo hi] [--sass]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[2]
stall = [(i, x) for i, x in enumerate(h) if x.startswith('stall_') and 'Not Issued' not in x]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 and sys.argv[2].isdigit() else (0, 10 ** 9)
sass = '--sass' in sys.argv


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


cur = None
for r in rows[3:]:
    if len(r) < 40:
        continue
    if r[0] != '':
        cur = num(r[0])
        if lo <= cur <= hi and (num(r[4]) or num(r[7])):
            st = sorted(((num(r[i]), n[6:]) for i, n in stall), reverse=True)[:4]
            print(f"{r[0]:>4} samp {num(r[4]):5d} inst {num(r[7]):9d} {' '.join(f'{n}={v}' for v, n in st if v)} | {r[1][:80]}")
    elif sass and cur is not None and lo <= cur <= hi and num(r[4]):
        st = sorted(((num(r[i]), n[6:]) for i, n in stall), reverse=True)[:3]
        print(f"        {r[3][:60]:60s} samp {num(r[4]):5d} {' '.join(f'{n}={v}' for v, n in st if v)}")
