"""Step time of one config under different L2 preparations (diagnostic): back-to-back steps on one
input set, a 256 MB write flush before each step, and a write flush followed by a 256 MB read."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2204_07143_b200 as na2d
from na2d_inputs import CONFIGS, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_ade20k_128"
s = CONFIGS[name]
inp = make_inputs(s, dtype="bf16", rpb="swin")
t = {n: torch.from_numpy(inp[n]).cuda().bfloat16() for n in ("q", "k", "v", "dout")}
rpb = torch.from_numpy(inp["rpb"]).cuda()
L = s.kernel_size
wbuf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(64 << 20, dtype=torch.float32, device="cuda")


def step():
    out, lse = na2d.forward(t["q"], t["k"], t["v"], rpb, L)
    na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], L)


for mode in ("back_to_back", "write_flush", "write_read_flush", "read_flush"):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    na2d.na2d_profile_enable(True)
    times = []
    for i in range(10):
        if mode in ("write_flush", "write_read_flush"):
            wbuf.fill_(i & 0xff)
        if mode in ("write_read_flush", "read_flush"):
            rbuf.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    prof = na2d.na2d_profile_read()
    na2d.na2d_profile_enable(False)
    print(mode, "ms/step", round(sorted(times)[5], 4), {k: round(1e3 * v[0] / v[1], 1) for k, v in prof.items()}, flush=True)
