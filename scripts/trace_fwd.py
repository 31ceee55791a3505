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
buf = torch.zeros(4 * 32 * 16, dtype=torch.int64, device="cuda")
for _ in range(2):
    na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
na2d.load_library().na2d_debug_set_trace(buf.data_ptr())
na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
torch.cuda.synchronize()
na2d.load_library().na2d_debug_set_trace(None)
tr = buf.cpu().numpy().reshape(4, 32, 16)
names = ["tma_issue", "mma_full_ok", "mma_tfree_ok", "mma_pfull_ok", "sm_wait_s", "sm_s_ok", "sm_pass1", "sm_pfull", "sm_o_ok", "sm_epi_done", "pf_q0", "pf_q1", "pf_q2", "pf_q3", "p2_wst"]
for cta in range(1):
    base = tr[cta][tr[cta] > 0].min()
    print(f"CTA {cta}")
    for it in range(8, 14):
        row = tr[cta, it]
        print(f"  tile {it:2d} " + " ".join(f"{n}={(row[e]-base) if row[e] else -1:7d}" for e, n in enumerate(names)))
