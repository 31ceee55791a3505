"""Multi-head neighborhood attention (MHNA) on top of the NA2D C ABI.

``NA2DFunction`` makes the library's forward / backward a ``torch.autograd.Function``;
``NeighborhoodAttention2D`` is the NAT attention layer around it:
a QKV linear, NA over every head with its relative positional bias, an output projection.
The linears are torch (cuBLAS) GEMMs -- "the steps either side of the path"; every NA step
runs in ``libna2d.so``.  There is no fallback: CPU tensors raise in the binding.

Bias convention: Eq. 2 literal (reading R1), ``s = scale * (q.k + B)``.  The layer's
``rpb`` parameter is that ``B``; a Swin-style table ``B_swin`` (added after scaling) corresponds
to ``B = B_swin / scale``.
"""
from __future__ import annotations

import math

import torch
from torch import nn

from . import backward as _na_backward
from . import forward as _na_forward


class NA2DFunction(torch.autograd.Function):
    """out = NA2D(q, k, v; rpb) on [B, heads, H, W, d] tensors (bf16 or fp32, CUDA)."""

    @staticmethod
    def forward(ctx, q, k, v, rpb, kernel_size: int, scale: float):
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        rpb_c = None if rpb is None else rpb.detach().float().contiguous()
        out, lse = _na_forward(q, k, v, rpb_c, kernel_size, scale)
        ctx.save_for_backward(q, k, v, rpb_c if rpb_c is not None else torch.empty(0, device=q.device), out, lse)
        ctx.has_rpb = rpb is not None
        ctx.rpb_dtype = None if rpb is None else rpb.dtype
        ctx.kernel_size, ctx.scale = kernel_size, scale
        return out

    @staticmethod
    def backward(ctx, dout):
        q, k, v, rpb, out, lse = ctx.saved_tensors
        rpb = rpb if ctx.has_rpb else None
        dq, dk, dv, drpb = _na_backward(q, k, v, rpb, out, lse, dout.contiguous(), ctx.kernel_size, ctx.scale)
        if drpb is not None:
            drpb = drpb.to(ctx.rpb_dtype)
        return dq, dk, dv, drpb, None, None


def na2d(q, k, v, rpb=None, kernel_size: int = 7, scale: float | None = None):
    """Differentiable NA2D (Eq. 2) on [B, heads, H, W, d] CUDA tensors."""
    if scale is None:
        scale = q.shape[-1] ** -0.5
    return NA2DFunction.apply(q, k, v, rpb, kernel_size, float(scale))


class NeighborhoodAttention2D(nn.Module):
    """NAT's neighborhood attention layer on channels-last maps [B, H, W, C].

    C = heads * head_dim; the relative positional bias table is [heads, 2k-1, 2k-1],
    initialised trunc-normal(0, 0.02) and scaled to the Eq. 2 convention.
    """

    def __init__(self, dim: int, heads: int, kernel_size: int = 7, qkv_bias: bool = True, rpb: bool = True,
                 dtype=torch.bfloat16, device=None):
        super().__init__()
        if dim % heads:
            raise ValueError(f"dim {dim} is not a multiple of heads {heads}")
        if kernel_size < 3 or kernel_size % 2 == 0:
            raise ValueError(f"kernel_size must be odd and >= 3 (P:438), got {kernel_size}")
        self.dim, self.heads, self.kernel_size = dim, heads, kernel_size
        self.head_dim = dim // heads
        self.scale = self.head_dim ** -0.5
        self.qkv = nn.Linear(dim, 3 * dim, bias=qkv_bias, dtype=dtype, device=device)
        self.proj = nn.Linear(dim, dim, dtype=dtype, device=device)
        if rpb:
            t = 2 * kernel_size - 1
            table = torch.empty(heads, t, t, dtype=torch.float32, device=device)
            nn.init.trunc_normal_(table, std=0.02, a=-2.0, b=2.0)
            self.rpb = nn.Parameter(table / self.scale)  # Eq. 2 convention (R1)
        else:
            self.register_parameter("rpb", None)

    def forward(self, x):
        b, h, w, c = x.shape
        qkv = self.qkv(x).view(b, h, w, 3, self.heads, self.head_dim).permute(3, 0, 4, 1, 2, 5)
        q, k, v = qkv[0], qkv[1], qkv[2]  # [B, heads, H, W, d]
        o = na2d(q, k, v, self.rpb, self.kernel_size, self.scale)
        return self.proj(o.permute(0, 2, 3, 1, 4).reshape(b, h, w, c))


class NATBlock(nn.Module):
    """One NAT block (Fig. 5): x + MHNA(LN(x)), then x + MLP(LN(x)); channels-last."""

    def __init__(self, dim: int, heads: int, kernel_size: int = 7, mlp_ratio: float = 3.0, dtype=torch.bfloat16,
                 device=None):
        super().__init__()
        self.norm1 = nn.LayerNorm(dim, dtype=dtype, device=device)
        self.attn = NeighborhoodAttention2D(dim, heads, kernel_size, dtype=dtype, device=device)
        self.norm2 = nn.LayerNorm(dim, dtype=dtype, device=device)
        hidden = int(math.ceil(dim * mlp_ratio))
        self.mlp = nn.Sequential(nn.Linear(dim, hidden, dtype=dtype, device=device), nn.GELU(),
                                 nn.Linear(hidden, dim, dtype=dtype, device=device))

    def forward(self, x):
        x = x + self.attn(self.norm1(x))
        return x + self.mlp(self.norm2(x))
