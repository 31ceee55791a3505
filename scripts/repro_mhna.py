"""Repro: an NA2D call, then the autograd bf16 grads test shape."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2204_07143_b200 as na2d
from paper_2204_07143_b200.mhna import na2d as na2d_fn
from na2d_inputs import Shape, make_inputs, CONFIGS
from tests.parity import run_cuda
first = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
if first == "host":
    import tests.test_gpu_parity as tg
    tg.test_step_host_matches_device_path()
    print("step_host ok")
if first == "cfg1":
    inp = make_inputs(CONFIGS["cfg1_8x8_k3"], seed=1)
    run_cuda(inp, 3, 32 ** -0.5, "bf16")
    print("cfg1 ok")
s = Shape("fn", 2, 2, 13, 18, 32, 7)
inp = make_inputs(s, seed=5, dtype="bf16")
t = {n: torch.from_numpy(inp[n]).cuda().to(torch.bfloat16).requires_grad_(n != "dout") for n in ("q", "k", "v", "dout")}
rpb = torch.from_numpy(inp["rpb"]).cuda().requires_grad_(True)
out = na2d_fn(t["q"], t["k"], t["v"], rpb, 7)
torch.cuda.synchronize()
print("fwd ok")
try:
    out.backward(t["dout"])
    torch.cuda.synchronize()
    print("bwd ok")
except Exception as e:
    print("bwd failed:", e)
    # direct call with explicit contiguous copies
    q, k, v = (x.detach().contiguous() for x in (t["q"], t["k"], t["v"]))
    o, lse = na2d.forward(q, k, v, rpb.detach(), 7)
    try:
        na2d.backward(q, k, v, rpb.detach(), o, lse, t["dout"].contiguous(), 7)
        torch.cuda.synchronize()
        print("direct bwd ok")
    except Exception as e2:
        print("direct bwd failed:", e2)
    for n in ("q", "k", "v", "dout"):
        print(n, t[n].data_ptr() % 1024, t[n].stride())
    print("dout", t["dout"].shape, t["dout"].stride(), t["dout"].dtype, t["dout"].data_ptr() % 256)
