"""B1 prologue / epilogue wall-clock breakdown (-DNA2D_TRACE build) on a problem with n tiles per
CTA (24 x 32 maps, 6 tiles each): entry -> after griddepcontrol.wait -> first bias table built ->
first S / dP landed -> loop end -> dRPB flush + commit done -> exit, for CTAs 0, 37, 74, 111."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2204_07143_b200 as na2d

per_cta = int(sys.argv[1]) if len(sys.argv) > 1 else 1
maps = 148 * per_cta // 6 + 1
B, heads, H, W = maps, 1, 24, 32
q, k, v, do = (torch.randn(B, heads, H, W, 32, device="cuda").bfloat16() for _ in range(4))
rpb = torch.randn(heads, 13, 13, device="cuda") * 0.02
out, lse = na2d.forward(q, k, v, rpb, 7)
for _ in range(3):
    na2d.backward(q, k, v, rpb, out, lse, do, 7)
buf = torch.zeros(24000, dtype=torch.int64, device="cuda")
lib = na2d.load_library()
torch.cuda.synchronize()
lib.na2d_debug_set_trace(buf.data_ptr())
na2d.backward(q, k, v, rpb, out, lse, do, 7)
torch.cuda.synchronize()
lib.na2d_debug_set_trace(None)
b = buf.cpu().numpy()
names = {16: "entry", 19: "pdl_ok", 20: "table", 21: "sp_ok", 17: "loop_end", 22: "ew_end", 23: "commit", 18: "exit"}
for cta in range(4):
    row = b[4096 + cta * 32 * 32: 4096 + cta * 32 * 32 + 32]
    t0 = row[16]
    print(f"CTA {cta * 37}: " + " ".join(f"{n}={(row[s] - t0) / 1e3:.2f}" for s, n in names.items() if row[s]))
# forward: trace[18000 + 8 cta + k]: entry, after griddepcontrol.wait, group-0 table built, first S
# landed, loop end, exit
buf.zero_()
lib.na2d_debug_set_trace(buf.data_ptr())
na2d.forward(q, k, v, rpb, 7)
torch.cuda.synchronize()
lib.na2d_debug_set_trace(None)
b = buf.cpu().numpy()
fn = ["entry", "pdl_ok", "table", "s_ok", "loop_end", "exit"]
for cta in (0, 37, 74, 111):
    row = b[18000 + 8 * cta: 18000 + 8 * cta + 6]
    print(f"fwd CTA {cta}: " + " ".join(f"{n}={(row[i] - row[0]) / 1e3:.2f}" for i, n in enumerate(fn) if row[i]))
# B1 tile-0 events of CTA 0 (clock64 cycles, relative to the MMA warp seeing the stage full)
buf.zero_()
lib.na2d_debug_set_trace(buf.data_ptr())
na2d.backward(q, k, v, rpb, out, lse, do, 7)
torch.cuda.synchronize()
lib.na2d_debug_set_trace(None)
b = buf.cpu().numpy()
ev = {0: "full", 2: "sp_iss", 3: "ds_seen", 1: "tfree", 4: "dq_iss", 8: "ew_w", 9: "sp_ok", 10: "p1", 11: "p2",
      12: "dq_ok", 13: "acc_rd", 14: "stored"}
for cta in (0, 37):
    row = b[4096 + (cta // 37) * 32 * 32: 4096 + (cta // 37) * 32 * 32 + 32]
    print(f"B1 CTA {cta} tile 0 (cycles from 'full'): " + " ".join(f"{n}={row[e] - row[0]}" for e, n in ev.items() if row[e]))
# B2: trace[19200 + 8 cta + k]: entry, after griddepcontrol.wait, dRPB sum done, first table, first
# S^T landed, loop end, exit
buf.zero_()
lib.na2d_debug_set_trace(buf.data_ptr())
na2d.backward(q, k, v, rpb, out, lse, do, 7)
torch.cuda.synchronize()
lib.na2d_debug_set_trace(None)
b = buf.cpu().numpy()
kn = ["entry", "pdl_ok", "drpb_sum", "table", "s_ok", "loop_end", "exit"]
for cta in (0, 37, 74, 111):
    row = b[19200 + 8 * cta: 19200 + 8 * cta + 7]
    print(f"B2 CTA {cta}: " + " ".join(f"{n}={(row[i] - row[0]) / 1e3:.2f}" for i, n in enumerate(kn) if row[i]))
