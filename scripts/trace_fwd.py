"""Dump the forward kernel's pipeline timeline (na2d_debug_set_trace) for cfg2."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from na2d_inputs import CONFIGS, make_inputs
import paper_2204_07143_b200 as na2d
s = CONFIGS["cfg2_nat_tiny_s1"]
inp = make_inputs(s, dtype="bf16", rpb="swin")
t = {n: torch.from_numpy(inp[n]).cuda().bfloat16() for n in ("q", "k", "v")}
rpb = torch.from_numpy(inp["rpb"]).cuda()
buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
for _ in range(2):
    na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
na2d.load_library().na2d_debug_set_trace(buf.data_ptr())
na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
torch.cuda.synchronize()
na2d.load_library().na2d_debug_set_trace(None)
full = buf.cpu().numpy()
if full[5000] > 0: print('MMA probe cycles per tile [plain, +wait, +fence, +both] CTA0..1:', full[5000:5008] / 20)
tr = full[:4096].reshape(4, 32, 32)
names = ["tma_issue", "mma_full_ok", "mma_tfree_ok", "mma_pv_done", "sm_wait_s", "sm_s_ok", "sm_pass1", "sm_pass2", "sm_o_ok", "sm_epi_done", "p2q0", "p2q1", "p2q2", "p2q3", "p1q0", "p1q1", "p1q2", "p1q3", "x", "mma_p0", "mma_p1", "mma_p2", "mma_p3", "mma_p4", "q0_p0", "q0_p1", "q0_p2", "q0_p3", "q0_p4", "x2", "mma_qk_issued"]
for cta in range(1):
    base = tr[cta][tr[cta] > 0].min()
    print(f"CTA {cta}")
    for it in range(8, 12):
        row = tr[cta, it]
        print(f"  tile {it:2d} " + " ".join(f"{n}={(row[e]-base) if row[e] else -1:6d}" for e, n in enumerate(names)))
