"""Step time of the CUDA-core (SIMT) path: fp32 I/O at NAT-Tiny stage-1 shape, and bf16 at d = 128 /
L = 9 (the shapes the tcgen05 kernels do not cover).  usage: simt_timing.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2204_07143_b200 as na2d


def run(B, heads, H, W, d, L, dtype, steps=5):
    q, k, v, do = (torch.randn(B, heads, H, W, d, device="cuda", dtype=dtype) for _ in range(4))
    rpb = torch.randn(heads, 2 * L - 1, 2 * L - 1, device="cuda") * 0.02
    out, lse = na2d.forward(q, k, v, rpb, L)
    na2d.backward(q, k, v, rpb, out, lse, do, L)
    torch.cuda.synchronize()
    na2d.na2d_profile_enable(True)
    for _ in range(steps):
        out, lse = na2d.forward(q, k, v, rpb, L)
        na2d.backward(q, k, v, rpb, out, lse, do, L)
    torch.cuda.synchronize()
    prof = na2d.na2d_profile_read()
    na2d.na2d_profile_enable(False)
    nq = B * heads * H * W
    fl = 12 * nq * min(L, H) * min(L, W) * d
    tot = sum(v[0] for v in prof.values()) / steps
    print(f"B={B} heads={heads} {H}x{W} d={d} L={L} {dtype}: {tot:.2f} ms/step, {fl / tot / 1e9:.2f} TFLOP/s",
          {k2: round(v2[0] / v2[1], 3) for k2, v2 in prof.items()}, flush=True)


run(128, 2, 56, 56, 32, 7, torch.float32)
run(16, 2, 56, 56, 128, 7, torch.bfloat16)
run(16, 2, 56, 56, 32, 9, torch.bfloat16)
