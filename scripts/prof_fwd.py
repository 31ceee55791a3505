"""Run forward (and optionally backward) on a BASELINE config a few times (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from na2d_inputs import CONFIGS, make_inputs
import paper_2204_07143_b200 as na2d
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_nat_tiny_s1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
bwd = "--bwd" in sys.argv
s = CONFIGS[name]
inp = make_inputs(s, dtype="bf16", rpb="swin")
t = {n: torch.from_numpy(inp[n]).cuda().bfloat16() for n in ("q", "k", "v", "dout")}
rpb = torch.from_numpy(inp["rpb"]).cuda()
for _ in range(reps):
    out, lse = na2d.forward(t["q"], t["k"], t["v"], rpb, s.kernel_size)
    if bwd:
        na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], s.kernel_size)
torch.cuda.synchronize()
print("done")
