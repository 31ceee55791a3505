"""B1 (dQ kernel) per-tile timeline of CTA 0 for cfg2 (build with -DNA2D_TRACE)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2204_07143_b200 as na2d
from na2d_inputs import CONFIGS, make_inputs

s = CONFIGS["cfg2_nat_tiny_s1"]
inp = make_inputs(s, dtype="bf16", rpb="swin")
t = {n: torch.from_numpy(inp[n]).cuda().bfloat16() for n in ("q", "k", "v", "dout")}
rpb = torch.from_numpy(inp["rpb"]).cuda()
out, lse = na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
buf = torch.zeros(32768 + 16 * 64 * 16 + 65536, dtype=torch.int64, device="cuda")
for _ in range(2):
    na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
na2d.load_library().na2d_debug_set_trace(buf.data_ptr())
na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
torch.cuda.synchronize()
na2d.load_library().na2d_debug_set_trace(None)
tr = buf.cpu().numpy()[32768:32768 + 16 * 64 * 16].reshape(16, 64, 16)
base = tr[tr > 0].min()
rel = np.where(tr > 0, tr - base, -1)
names = {0: "start", 1: "p1f0", 2: "p1f1", 3: "pfr0", 4: "pfr1", 5: "Dbar", 6: "epi", 7: "p2f0", 8: "p2f1", 9: "ds0", 10: "ds1"}
for it in range(4, 9):
    print(f"--- tile {it}: producer empty_ok={rel[12, it, 0]}")
    print("  issA S/dP1 issue:", [int(x) for x in rel[13, it, :5]])
    print("  issB dP2 issue:  ", [int(x) for x in rel[14, it, :5]])
    print("  issC dQ issue:   ", [int(x) for x in rel[15, it, :5]])
    for g in range(3):
        w = 4 * g
        print(f"  grp{g}: " + " ".join(f"{n}={rel[w, it, e]}" for e, n in names.items() if rel[w, it, e] >= 0))
d = rel[0, 5:40, 0] - rel[0, 4:39, 0]
print("tile period (grp0 start) median", np.median(d[d > 0]))
