"""Where are the largest dQ errors?  cfg2 B=4 vs the fp64 oracle, by position."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from na2d_inputs import CONFIGS, make_inputs
from tests.parity import run_cuda, run_oracle
s = CONFIGS["cfg2_nat_tiny_s1"].replace(B=4)
inp = make_inputs(s, seed=5)
got = run_cuda(inp, 7, 32 ** -0.5, "bf16")
ref = run_oracle(inp, 7, 32 ** -0.5)
for n in ("dq", "dk", "dv"):
    e = np.abs(got[n] - ref[n]).max(-1)  # [B,h,H,W]
    flat = np.argsort(e.ravel())[::-1][:8]
    locs = [np.unravel_index(f, e.shape) for f in flat]
    print(n, "max", e.max(), "mean", e.mean(), "top", [(int(a[2]), int(a[3]), round(float(e[a]), 4)) for a in locs])
    byrow = e.mean(axis=(0, 1, 3)); bycol = e.mean(axis=(0, 1, 2))
    print("  mean err by row", np.round(byrow[:12] * 1e3, 2), "...", np.round(byrow[-8:] * 1e3, 2))
    print("  mean err by row%8", [round(float(e[:, :, r::8].mean()) * 1e3, 3) for r in range(8)])
    print("  mean err by col%16", [round(float(e[:, :, :, c::16].mean()) * 1e3, 3) for c in range(16)])
