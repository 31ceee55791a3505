"""Per-CTA wall-clock spans of the three kernels at cfg2 (builds with -DNA2D_TRACE): load balance."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from na2d_inputs import CONFIGS, make_inputs
import paper_2204_07143_b200 as na2d
s = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2_nat_tiny_s1"]
inp = make_inputs(s, dtype="bf16", rpb="swin")
t = {n: torch.from_numpy(inp[n]).cuda().bfloat16() for n in ("q", "k", "v", "dout")}
rpb = torch.from_numpy(inp["rpb"]).cuda()
for _ in range(2):
    out, lse = na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
    na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
buf = torch.zeros(24000, dtype=torch.int64, device="cuda")
lib = na2d.load_library()
lib.na2d_debug_set_trace(buf.data_ptr())
out, lse = na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
torch.cuda.synchronize()
lib.na2d_debug_set_trace(None)
b = buf.cpu().numpy()
for name, off in (("fwd", 16384), ("B1", 16384 + 512), ("B2", 16384 + 1024)):
    st, en = b[off:off + 296:2], b[off + 1:off + 297:2]
    ok = (st > 0) & (en > 0)
    st, en = st[ok], en[ok]
    if not ok.any():
        print(f"{name}: no span recorded")
        continue
    t0 = st.min()
    dur = (en - st) / 1e3
    print(f"{name}: CTAs {ok.sum()}  kernel span {(en.max() - t0) / 1e3:.1f} us  start spread {(st.max() - t0) / 1e3:.1f} us  "
          f"CTA duration min/median/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us  end spread {(en.max() - en.min()) / 1e3:.1f} us")
    order = np.argsort(en)
    print("   slowest CTAs:", order[-5:], "fastest:", order[:5])
# B1 per-CTA durations in CTA order (contiguous tile ranges of the class-grouped order)
off = 16384 + 512
st, en = b[off:off + 296:2], b[off + 1:off + 297:2]
dur = (en - st) / 1e3
print("B1 per-CTA duration (us), CTA 0..147:")
print(" ".join(f"{x:.0f}" for x in dur))
