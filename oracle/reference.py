"""Independent NumPy / PyTorch-CPU formulations of 2D Neighborhood Attention.

TEST INFRASTRUCTURE ONLY (same import rule as the ``oracle`` package).  These exist to pin
the C oracle against formulations that share none of its code or index arithmetic:

* ``window_start_argmin``  -- rho as "the window whose centre is nearest the query"
  ("pixels nearest to (i,j)", "continuing to pick the L^2 nearest"), found by
  brute-force argmin over all window positions; no clamp formula.
* ``unfold_windows``       -- Appendix A: stride-1 sliding-window extraction
  ("unfold") followed by replicate padding of the extracted windows ("replicated_pad").
* ``na2d_unfold_forward``  -- Eq. 2 evaluated on the unfolded K/V tensors, with the
  relative-position bias looked up through unfolded coordinate grids.
* ``na2d_dense``           -- Eq. 1 dense self-attention over all H*W tokens with an
  additive mask/bias matrix built by brute-force enumeration from ``window_start_argmin``;
  differentiable through torch.autograd (fp64) for an independent gradient check.
"""
from __future__ import annotations

import numpy as np


def window_start_argmin(i: int, n: int, L: int) -> int:
    """Start of the length-min(L,n) window whose centre is nearest to i (unique: centres are
    consecutive integers and i is an integer, so no ties)."""
    if L >= n:
        return 0
    half = (L - 1) // 2
    best, best_dist = None, None
    for s in range(0, n - L + 1):
        dist = abs(s + half - i)
        if best_dist is None or dist < best_dist:
            best, best_dist = s, dist
    return best


def unfold_windows(x: np.ndarray, L: int) -> np.ndarray:
    """Appendix A: x [H, W, C] -> [H, W, Lh, Lw, C].

    'unfold' with stride 1 gives one window per position where a full window fits; the
    extracted window tensor is then replicate-padded along the two position axes so the
    border pixels reuse the nearest full window.  An axis shorter than L uses the whole
    axis as its (single) window."""
    H, W, C = x.shape
    Lh, Lw = min(L, H), min(L, W)
    nh, nw = H - Lh + 1, W - Lw + 1
    win = np.empty((nh, nw, Lh, Lw, C), dtype=x.dtype)
    for a in range(nh):            # unfold, stride 1
        for b in range(nw):
            win[a, b] = x[a:a + Lh, b:b + Lw]
    ph, pw = (H - nh), (W - nw)   # replicate pad to H x W positions, (L-1)/2 per side
    top, left = ph // 2, pw // 2
    pad = ((top, ph - top), (left, pw - left), (0, 0), (0, 0), (0, 0))
    return np.pad(win, pad, mode="edge")


def na2d_unfold_forward(q, k, v, rpb, L: int, inv_scale: float):
    """Eq. 2 on unfold+replicate-pad neighbourhoods.  q,k,v: [B,heads,H,W,d] -> (out, lse)."""
    q, k, v = (np.asarray(t, np.float64) for t in (q, k, v))
    B, heads, H, W, d = q.shape
    rows = np.broadcast_to(np.arange(H, dtype=np.float64)[:, None, None], (H, W, 1))
    cols = np.broadcast_to(np.arange(W, dtype=np.float64)[None, :, None], (H, W, 1))
    prow = unfold_windows(np.ascontiguousarray(rows), L)[..., 0].astype(int)  # key row of window entry
    pcol = unfold_windows(np.ascontiguousarray(cols), L)[..., 0].astype(int)
    ii = np.arange(H)[:, None, None, None]
    jj = np.arange(W)[None, :, None, None]
    out = np.empty_like(q)
    lse = np.empty(q.shape[:4])
    for b in range(B):
        for h in range(heads):
            Kw = unfold_windows(k[b, h], L)  # [H,W,Lh,Lw,d]
            Vw = unfold_windows(v[b, h], L)
            dots = np.einsum("ijc,ijabc->ijab", q[b, h], Kw)
            bias = 0.0
            if rpb is not None:
                bias = np.asarray(rpb, np.float64)[h][prow - ii + L - 1, pcol - jj + L - 1]
            s = inv_scale * (dots + bias)
            m = s.max(axis=(2, 3), keepdims=True)
            e = np.exp(s - m)
            z = e.sum(axis=(2, 3), keepdims=True)
            p = e / z
            out[b, h] = np.einsum("ijab,ijabc->ijc", p, Vw)
            lse[b, h] = (m + np.log(z))[..., 0, 0]
    return out, lse


def neighbourhood_bias_matrix(H: int, W: int, L: int, table=None) -> np.ndarray:
    """[H*W, H*W] additive matrix: table[key-query+L-1] on pairs with key in rho(query) found
    by brute-force enumeration (window_start_argmin), -inf elsewhere."""
    M = np.full((H * W, H * W), -np.inf)
    for i in range(H):
        si, li = window_start_argmin(i, H, L), min(L, H)
        for j in range(W):
            sj, lj = window_start_argmin(j, W, L), min(L, W)
            for p in range(si, si + li):
                for qq in range(sj, sj + lj):
                    M[i * W + j, p * W + qq] = 0.0 if table is None else table[p - i + L - 1, qq - j + L - 1]
    return M


def na2d_dense(q, k, v, rpb, L: int, inv_scale: float):
    """Eq. 1 dense attention over all H*W tokens + the brute-force neighbourhood mask/bias,
    in torch fp64 (CPU).  Accepts torch tensors (may require grad) -> (out, lse) tensors."""
    import torch

    B, heads, H, W, d = q.shape
    outs, lses = [], []
    for h in range(heads):
        if rpb is None:
            add = torch.from_numpy(neighbourhood_bias_matrix(H, W, L))
        else:
            mask = torch.from_numpy(neighbourhood_bias_matrix(H, W, L))
            # gather the table through an index map so gradients flow to rpb
            idx = np.zeros((H * W, H * W), dtype=np.int64)
            T = 2 * L - 1
            for i in range(H):
                for j in range(W):
                    for p in range(H):
                        for qq in range(W):
                            a, c = p - i + L - 1, qq - j + L - 1
                            idx[i * W + j, p * W + qq] = (a * T + c) if (0 <= a < T and 0 <= c < T) else 0
            add = rpb[h].reshape(-1)[torch.from_numpy(idx)]
            add = torch.where(torch.isinf(mask), mask, add)
        qh = q[:, h].reshape(B, H * W, d)
        kh = k[:, h].reshape(B, H * W, d)
        vh = v[:, h].reshape(B, H * W, d)
        s = inv_scale * (qh @ kh.transpose(1, 2) + add)
        lse = torch.logsumexp(s, dim=-1)
        p = torch.exp(s - lse[..., None])
        outs.append((p @ vh).reshape(B, H, W, d))
        lses.append(lse.reshape(B, H, W))
    return torch.stack(outs, 1), torch.stack(lses, 1)


def self_attention(q, k, v):
    """Eq. 1: softmax(Q K^T / sqrt(d_k)) V over M tokens.  q,k,v: [M, d] fp64."""
    q, k, v = (np.asarray(t, np.float64) for t in (q, k, v))
    s = q @ k.T / np.sqrt(q.shape[-1])
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=-1, keepdims=True)
    return p @ v
