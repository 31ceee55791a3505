"""Dump the forward kernel's pipeline timeline (na2d_debug_set_trace; library built with
NA2D_NVCC_EXTRA=-DNA2D_TRACE) for cfg2: per tile, SM cycles of each event."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from na2d_inputs import CONFIGS, make_inputs
import paper_2204_07143_b200 as na2d
s = CONFIGS["cfg2_nat_tiny_s1"]
inp = make_inputs(s, dtype="bf16", rpb="swin")
t = {n: torch.from_numpy(inp[n]).cuda().bfloat16() for n in ("q", "k", "v")}
rpb = torch.from_numpy(inp["rpb"]).cuda()
buf = torch.zeros(8192 * 4, dtype=torch.int64, device="cuda")
for _ in range(2):
    na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
na2d.load_library().na2d_debug_set_trace(buf.data_ptr())
na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
torch.cuda.synchronize()
na2d.load_library().na2d_debug_set_trace(None)
tr = buf.cpu().numpy()[:4 * 32 * 32].reshape(4, 32, 32)
names = {0: "tma", 1: "qk_full", 2: "qk_issue", 3: "pv_pready", 4: "pv_issue", 5: "ew_wait", 6: "ew_s", 7: "ew_max",
         9: "ew_pready", 10: "ew_oful", 12: "ew_ofree", 13: "ew_end"}
base = tr[0][tr[0] > 0].min()
for it in range(8, 14):
    row = tr[0, it]
    print(f"tile {it:2d} " + " ".join(f"{n}={(row[e] - base) if row[e] else -1:6d}" for e, n in names.items()))
ph = []
for cta in range(4):
    for it in range(4, 28):
        r = tr[cta, it]
        if r[13] == 0 or r[2] == 0:
            continue
        ph.append([r[2] - tr[cta, it - 1, 2], r[6] - r[2], r[6] - r[5], r[7] - r[6], r[9] - r[7], r[4] - r[9], r[10] - r[4],
                   r[12] - r[10], r[13] - r[12], r[5] - tr[cta, it - 2, 13] if it >= 2 and tr[cta, it - 2, 13] else 0])
print("median: period(QK issue), qk_issue->s_ok, ew wait for S, load+max, exp+store+sum, pready->pv_issue,"
      " pv_issue->o_full, o_full->o_free, stores, prev end->s_wait")
print(np.median(np.array(ph), axis=0))
