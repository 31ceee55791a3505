"""Per-launch fixed cost of the three tcgen05 kernels: per-kernel CUDA-event times (library
profiler) for n = 1, 2, 4, 8 tiles per CTA on a 24 x 32 map (3 x 2 tiles), B*heads scaled so
the grid stays at 148 CTAs; the intercept of time vs tiles-per-CTA is the fixed cost."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2204_07143_b200 as na2d

lib = na2d.load_library()
rows = []
for per_cta in (1, 2, 4, 8, 16):
    maps = 148 * per_cta // 6 + 1  # 6 tiles per 24 x 32 map
    B, heads, H, W = maps, 1, 24, 32
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn(B, heads, H, W, 32, device="cuda", generator=g).bfloat16() for _ in range(4))
    rpb = torch.randn(heads, 13, 13, device="cuda") * 0.02
    out, lse = na2d.forward(q, k, v, rpb, 7)
    grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty_like(rpb))
    for _ in range(3):
        na2d.backward(q, k, v, rpb, out, lse, do, 7)
    torch.cuda.synchronize()
    na2d.na2d_profile_enable(True)
    for _ in range(20):
        out, lse = na2d.forward(q, k, v, rpb, 7)
        na2d.backward(q, k, v, rpb, out, lse, do, 7)
    torch.cuda.synchronize()
    prof = na2d.na2d_profile_read()
    na2d.na2d_profile_enable(False)
    t = {kk: vv[0] / vv[1] * 1e3 for kk, vv in prof.items()}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        out, lse = na2d.forward(q, k, v, rpb, 7, out=out, lse=lse)
        na2d.backward(q, k, v, rpb, out, lse, do, 7, grads=grads)
    e1.record()
    torch.cuda.synchronize()
    t["step (no events)"] = e0.elapsed_time(e1) / 20 * 1e3
    rows.append((maps * 6 / 148, t))
    print(f"tiles/CTA {maps * 6 / 148:5.2f}", {kk: round(vv, 1) for kk, vv in t.items()})
for name in rows[0][1]:
    x = np.array([r[0] for r in rows]); y = np.array([r[1][name] for r in rows])
    a, b = np.polyfit(x, y, 1)
    print(f"{name}: {a:.2f} us per tile per CTA, fixed {b:.1f} us")
