"""Timeline of the two-stream B1 (CTA 0) at cfg2; build with -DNA2D_TRACE."""
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
buf = torch.zeros(32768 + 24 * 64 * 16 + 65536, dtype=torch.int64, device="cuda")
for _ in range(2):
    na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
na2d.load_library().na2d_debug_set_trace(buf.data_ptr())
na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
torch.cuda.synchronize()
na2d.load_library().na2d_debug_set_trace(None)
nw = int(sys.argv[1]) if len(sys.argv) > 1 else 11
tr = buf.cpu().numpy()[32768:32768 + 24 * 64 * 16].reshape(24, 64, 16)[:nw]
base = tr[tr > 0].min()
rel = np.where(tr > 0, tr - base, -1)
mma0, mma1 = nw - 2, nw - 1
for it in range(4, 9):
    print(f"--- tile {it}")
    for sm, w in ((0, mma0), (1, mma1)):
        print(f"  mma{sm}: full={rel[w, it, 0]} sdp_iss={rel[w, it, 1]} ds_seen={rel[w, it, 2]} dqfree={rel[w, it, 3]} dq_iss={rel[w, it, 4]}")
    for w in (0, 4):
        print(f"  ew{w}: wait={rel[w, it, 5]} sp_ok={rel[w, it, 6]} p1={rel[w, it, 7]} D={rel[w, it, 8]} p2={rel[w, it, 9]}")
d = rel[0, 5:40, 6] - rel[0, 4:39, 6]
print("stream-0 period median", np.median(d[d > 0]))
