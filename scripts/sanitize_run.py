"""Small forward + backward of every library path under compute-sanitizer (memcheck / racecheck /
synccheck): tcgen05 bf16 (k = 3, 5, 7, ragged maps, a row band), SIMT fp32, the paper's unfused
decomposition, and the pipelined host-buffer step.  Exits non-zero on a parity failure."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_07143_b200 as na2d  # noqa: E402
from na2d_inputs import Shape, make_inputs  # noqa: E402
from tests.parity import run_cuda  # noqa: E402

cases = [
    (Shape("s7", 2, 2, 19, 37, 32, 7), "bf16"),
    (Shape("s5", 1, 2, 13, 21, 32, 5), "bf16"),
    (Shape("s3", 1, 1, 9, 18, 32, 3), "bf16"),
    (Shape("f32", 1, 2, 11, 14, 32, 7), "f32"),
    (Shape("d16", 2, 2, 19, 37, 16, 7), "bf16"),  # tcgen05, 32-byte swizzled rows
    (Shape("d64", 2, 2, 19, 37, 64, 7), "bf16"),  # tcgen05, 128-byte rows, single stage, dQ in two passes
    (Shape("d64k5f16", 1, 2, 13, 21, 64, 5), "f16"),
    (Shape("d128", 1, 2, 11, 14, 128, 7), "bf16"),  # SIMT (incl. the fixed-order dRPB reduction)
    (Shape("pair7", 4, 3, 7, 7, 32, 7), "bf16"),  # small-map pair mode (two maps per tile, 5-D TMA views)
    (Shape("pair3", 4, 2, 3, 4, 32, 3), "f16"),
]
only = sys.argv[1:]  # optional case names (s7 s5 s3 f32 d16 d64 d64k5f16 d128 pair7 pair3 paper)
for s, dt in cases:
    if only and s.name not in only:
        continue
    inp = make_inputs(s, seed=3, dtype=dt)
    got = run_cuda(inp, s.kernel_size, s.d ** -0.5, dt)
    assert all(np.isfinite(v).all() for v in got.values()), s
    print("ok", s.name, dt, flush=True)
if only and "paper" not in only:
    sys.exit(0)
# the paper's decomposition
s = Shape("p", 1, 2, 12, 15, 32, 7)
inp = make_inputs(s, seed=4)
t = {n: torch.from_numpy(inp[n]).cuda().bfloat16() for n in ("q", "k", "v", "dout")}
rpb = torch.from_numpy(inp["rpb"]).cuda()
out, lse, attn = na2d.paper_forward(t["q"], t["k"], t["v"], rpb, 7, 32 ** -0.5)
na2d.paper_backward(t["q"], t["k"], t["v"], rpb, attn, t["dout"], 7, 32 ** -0.5)
torch.cuda.synchronize()
print("ok paper decomposition", flush=True)
