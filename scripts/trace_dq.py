"""Dump the B1 (dQ) kernel's per-tile pipeline timeline for cfg2 (CTA 0)."""
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
lib = na2d.load_library()
for _ in range(2):
    na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
# B1 runs first in the backward and B2 overwrites the buffer with its own events: trace B1 alone
# by enabling the buffer, running the backward, and reading B1's slots (B2 uses different CTAs'
# rows only where its chunk index < 32 -- so use a separate buffer per kernel: B1 first)
buf = torch.zeros(2 * 4 * 32 * 32, dtype=torch.int64, device="cuda")
lib.na2d_debug_set_trace(buf.data_ptr())
na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
torch.cuda.synchronize()
lib.na2d_debug_set_trace(None)
tr = buf.cpu().numpy()[4096:].reshape(4, 32, 32)
names = {0: "full", 1: "tfree", 2: "sp_iss", 3: "ds_seen", 4: "dq_iss", 8: "ew_w", 9: "sp_ok", 10: "p1", 11: "p2",
         12: "dq_ok", 13: "acc_rd", 14: "stored"}
cta = 0
base = tr[cta][tr[cta] > 0].min()
for it in range(2, 14):
    row = tr[cta, it]
    print(f"t{it:2d} " + " ".join(f"{n}={(row[e]-base) if row[e] else -1:6d}" for e, n in names.items()))
print("tile periods (full -> next full) per CTA:")
for cta in range(4):
    f = tr[cta, :, 0]
    d = [int(f[i + 1] - f[i]) for i in range(31) if f[i] and f[i + 1]]
    print(cta, d)
# effective clock: B1 event time vs traced cycles per tile (CTA 0), L2-hot and after an L2 flush
import numpy as np
per_tile = np.median([tr[0, i + 1, 0] - tr[0, i, 0] for i in range(31)])
ntiles = 128 * 2 * 7 * 4 / 148
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for cold in (False, True):
    lib.na2d_profile_enable(1)
    for _ in range(10):
        if cold:
            flush.zero_()
        na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)
    torch.cuda.synchronize()
    prof = na2d.na2d_profile_read()
    lib.na2d_profile_enable(0)
    ms = prof["na2d_bwd_dq_tc"][0] / prof["na2d_bwd_dq_tc"][1]
    print(f"cold={cold}: B1 {ms*1e3:.1f} us; traced {per_tile:.0f} cyc/tile x {ntiles:.1f} tiles -> "
          f"{per_tile*ntiles/(ms*1e-3)/1e9:.2f} GHz effective")
    print({k: round(v[0] / v[1] * 1e3, 1) for k, v in prof.items()})
for cta in range(4):
    c0, c1 = tr[cta, 0, 0], tr[cta, 31, 0]
    g0, g1 = tr[cta, 0, 15], tr[cta, 31, 15]
    print(f"CTA {cta*37}: {c1 - c0} cycles in {(g1 - g0)} ns -> {(c1 - c0) / (g1 - g0):.3f} GHz")
for cta in range(4):
    g = tr[cta, 0]
    print(f"CTA {cta*37}: entry->first full {(g[15]-g[16])} ns, entry->loop end {(g[17]-g[16])} ns, entry->exit {(g[18]-g[16])} ns")
