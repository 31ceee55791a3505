"""Size of the error D = dO . bf16(O) (instead of the exact dO . O) injects into dK and dQ, in fp64 numpy
on one batch of a BASELINE config (DESIGN round-2 table).  usage: d_error_bf16_out.py [config]
Prints per head: max |delta D|, max |delta dQ|, max |delta dK|, max |O|."""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from na2d_inputs import CONFIGS, make_inputs, bf16_round
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_ade20k_128"
s = CONFIGS[name]
inp = make_inputs(s, dtype="bf16", rpb="parity", batch_count=1)
L = s.kernel_size; H, W, d = s.H, s.W, s.d
scale = d ** -0.5
def ws(i, n):
    st = np.clip(i - (L - 1) // 2, 0, n - L); return st
si = ws(np.arange(H), H); sj = ws(np.arange(W), W)
worst = {}
for h in range(s.heads):
    q = inp["q"][0, h].astype(np.float64); k = inp["k"][0, h].astype(np.float64)
    v = inp["v"][0, h].astype(np.float64); do = inp["dout"][0, h].astype(np.float64)
    B = inp["rpb"][h].astype(np.float64)
    I = si[:, None, None, None] + np.arange(L)[None, None, :, None]  # [H,1,L,1]
    J = sj[None, :, None, None] + np.arange(L)[None, None, None, :]  # [1,W,1,L]
    I = np.broadcast_to(I, (H, W, L, L)); J = np.broadcast_to(J, (H, W, L, L))
    kw = k[I, J]; vw = v[I, J]   # [H,W,L,L,d]
    bi = I - np.arange(H)[:, None, None, None] + L - 1; bj = J - np.arange(W)[None, :, None, None] + L - 1
    s_ = scale * (np.einsum('ijd,ijabd->ijab', q, kw) + B[bi, bj])
    s_ = s_.reshape(H, W, L * L); s_ -= s_.max(-1, keepdims=True)
    P = np.exp(s_); P /= P.sum(-1, keepdims=True)
    O = np.einsum('ijn,ijnd->ijd', P, vw.reshape(H, W, L * L, d))
    dl = np.einsum('ijd,ijd->ij', do, bf16_round(O.astype(np.float32)).astype(np.float64) - O)
    # dQ change: -scale * dl * sum_k P k
    dq = -scale * dl[..., None] * np.einsum('ijn,ijnd->ijd', P, kw.reshape(H, W, L * L, d))
    # dK change: scatter -scale * P * dl * q onto keys
    dk = np.zeros_like(k)
    contrib = -scale * (P * dl[..., None])[..., None] * q[:, :, None, :]  # [H,W,49,d]
    np.add.at(dk, (I.reshape(H, W, -1), J.reshape(H, W, -1)), contrib)
    worst[h] = (np.abs(dl).max(), np.abs(dq).max(), np.abs(dk).max(), np.abs(O).max())
print(name, {h: tuple(round(float(x), 5) for x in w) for h, w in worst.items()})
