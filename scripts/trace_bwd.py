"""Dump the B2 (dK/dV) kernel's pipeline timeline for cfg2."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from na2d_inputs import CONFIGS, make_inputs
import paper_2204_07143_b200 as na2d
s = CONFIGS["cfg2_nat_tiny_s1"]
inp = make_inputs(s, dtype="bf16", rpb="swin")
t = {n: torch.from_numpy(inp[n]).cuda().bfloat16() for n in ("q", "k", "v", "dout")}
rpb = torch.from_numpy(inp["rpb"]).cuda()
out, lse = na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
buf = torch.zeros(2 * 4 * 32 * 32, dtype=torch.int64, device="cuda")
for _ in range(2):
    na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
na2d.load_library().na2d_debug_set_trace(buf.data_ptr())
na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
torch.cuda.synchronize()
na2d.load_library().na2d_debug_set_trace(None)
tr = buf.cpu().numpy()[:4096].reshape(4, 32, 32)
names = {0: "S_iss", 1: "ds_seen", 2: "kv_iss", 3: "full_ok", 4: "ew_wait", 5: "s_ok", 6: "ew_done", 7: "epi", 8: "acc_rd", 9: "stored", 10: "q0", 11: "q1", 12: "q2", 13: "q3", 16: "g0_top", 17: "g0_set", 18: "g0_full", 20: "g1_top", 21: "g1_set", 22: "g1_full"}
cta = 0
base = tr[cta][tr[cta] > 0].min()
for it in range(0, 8):
    print(f"tile {it}: producer empty_ok={tr[cta, it, 14]-base} staged={tr[cta, it, 15]-base}")
for c in range(4, 20):
    row = tr[cta, c]
    print(f"c{c:2d} " + " ".join(f"{n}={(row[e]-base) if row[e] else -1:6d}" for e, n in names.items()))
