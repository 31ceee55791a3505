"""Run forward + backward once on a (B, heads, H, W, L) problem and print max errors vs the oracle
when small enough (debug helper).  usage: one_case.py B heads H W L [--no-check]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2204_07143_b200 as na2d
from na2d_inputs import Shape, make_inputs

B, heads, H, W, L = (int(x) for x in sys.argv[1:6])
s = Shape("case", B, heads, H, W, 32, L)
inp = make_inputs(s, dtype="bf16", rpb="parity")
t = {n: torch.from_numpy(inp[n]).cuda().bfloat16() for n in ("q", "k", "v", "dout")}
rpb = torch.from_numpy(inp["rpb"]).cuda()
t0 = time.time()
out, lse = na2d.forward(t["q"], t["k"], t["v"], rpb, L)
g = na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], L)
torch.cuda.synchronize()
msg = f"B={B} heads={heads} {H}x{W} L={L}: {time.time() - t0:.2f}s"
if "--no-check" not in sys.argv and B * heads * H * W <= 200000:
    import oracle
    ref = oracle.na2d_backward(inp["q"], inp["k"], inp["v"], inp["rpb"], inp["dout"], L, 32 ** -0.5)
    for i, n in enumerate(("dq", "dk", "dv", "drpb")):
        msg += f" {n}={np.abs(g[i].float().cpu().numpy() - ref[n]).max():.4f}"
print(msg, flush=True)
