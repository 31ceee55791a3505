"""Neighborhood Attention Transformer (NAT) classification model around the NA2D kernels
(a full NAT forward as a workload-level benchmark).

Architecture as PAPER.md states it (§3.3 "Neighborhood Attention Transformer", P:204-224,
Table 2):
  * tokenizer: two consecutive 3x3 convolutions with 2x2 strides -> H/4 x W/4;
  * 4 levels of NAT blocks (x + MHNA(LN(x)), x + MLP(LN(x))), 7x7 neighbourhoods
    (Table 2 caption), every level but the last followed by a downsampler, a 3x3 stride-2
    convolution that halves the spatial size and doubles the channels;
  * dims and heads double after every level (Table 2 caption): level-1 dim = 32 x heads;
  * LayerScale for the larger models.
Readings where the paper is silent (R-NAT): the tokenizer's first convolution has
C/2 output channels; a LayerNorm follows the tokenizer and each downsampler; the classifier is
LN -> global average pool -> Linear(1000) (the usual hierarchical-transformer head); LayerScale
(init 1e-5) only where `layer_scale` is given.  With these readings the parameter and FLOP
counts reproduce Table 2 (tests/test_nat.py pins them: 20/28/51/90 M params,
2.7/4.3/7.8/13.7 GFLOPs at 224x224 counting multiply-accumulates).

Weights are random (no trained checkpoints exist here, SURVEY §2 out of scope); every NA step
runs in libna2d.so through ``mhna.na2d``; convolutions, LayerNorms and linears are torch.
"""
from __future__ import annotations

import math

import torch
from torch import nn

from .mhna import NATBlock

# Table 2: layers per level, level-1 heads (head dim 32), MLP ratio
VARIANTS = {
    "mini": dict(depths=(3, 4, 6, 5), heads=2, mlp_ratio=3.0),
    "tiny": dict(depths=(3, 4, 18, 5), heads=2, mlp_ratio=3.0),
    "small": dict(depths=(3, 4, 18, 5), heads=3, mlp_ratio=2.0),
    "base": dict(depths=(3, 4, 18, 5), heads=4, mlp_ratio=2.0),
}
HEAD_DIM = 32  # "32 x heads" (Table 2)


class ConvTokenizer(nn.Module):
    """Two 3x3 stride-2 convolutions, then LayerNorm; NCHW in, channels-last out."""

    def __init__(self, in_ch: int, dim: int, dtype, device):
        super().__init__()
        self.proj = nn.Sequential(
            nn.Conv2d(in_ch, dim // 2, 3, 2, 1, dtype=dtype, device=device),
            nn.Conv2d(dim // 2, dim, 3, 2, 1, dtype=dtype, device=device))
        self.norm = nn.LayerNorm(dim, dtype=dtype, device=device)

    def forward(self, x):
        return self.norm(self.proj(x).permute(0, 2, 3, 1))


class ConvDownsampler(nn.Module):
    """3x3 stride-2 convolution doubling the channels, then LayerNorm; channels-last."""

    def __init__(self, dim: int, dtype, device):
        super().__init__()
        self.reduction = nn.Conv2d(dim, 2 * dim, 3, 2, 1, bias=False, dtype=dtype, device=device)
        self.norm = nn.LayerNorm(2 * dim, dtype=dtype, device=device)

    def forward(self, x):
        return self.norm(self.reduction(x.permute(0, 3, 1, 2)).permute(0, 2, 3, 1))


class LayerScaleBlock(NATBlock):
    """NAT block with LayerScale: x + g1 * MHNA(LN(x)), x + g2 * MLP(LN(x))."""

    def __init__(self, dim, heads, kernel_size, mlp_ratio, layer_scale: float, dtype, device):
        super().__init__(dim, heads, kernel_size, mlp_ratio, dtype=dtype, device=device)
        self.gamma1 = nn.Parameter(torch.full((dim,), layer_scale, dtype=dtype, device=device))
        self.gamma2 = nn.Parameter(torch.full((dim,), layer_scale, dtype=dtype, device=device))

    def forward(self, x):
        x = x + self.gamma1 * self.attn(self.norm1(x))
        return x + self.gamma2 * self.mlp(self.norm2(x))


class NAT(nn.Module):
    """NAT classifier on NCHW images; NA2D runs on [B, heads, H, W, 32] per block."""

    def __init__(self, variant: str = "tiny", kernel_size: int = 7, in_ch: int = 3, num_classes: int = 1000,
                 layer_scale: float | None = None, dtype=torch.bfloat16, device=None):
        super().__init__()
        cfg = VARIANTS[variant]
        self.variant, self.kernel_size = variant, kernel_size
        heads = cfg["heads"]
        dim = heads * HEAD_DIM
        self.patch_embed = ConvTokenizer(in_ch, dim, dtype, device)
        self.levels = nn.ModuleList()
        self.downsamplers = nn.ModuleList()
        for lvl, depth in enumerate(cfg["depths"]):
            if layer_scale is None:
                blocks = [NATBlock(dim, heads, kernel_size, cfg["mlp_ratio"], dtype=dtype, device=device)
                          for _ in range(depth)]
            else:
                blocks = [LayerScaleBlock(dim, heads, kernel_size, cfg["mlp_ratio"], layer_scale, dtype, device)
                          for _ in range(depth)]
            self.levels.append(nn.Sequential(*blocks))
            if lvl < len(cfg["depths"]) - 1:
                self.downsamplers.append(ConvDownsampler(dim, dtype, device))
                dim, heads = 2 * dim, 2 * heads
        self.num_features = dim
        self.norm = nn.LayerNorm(dim, dtype=dtype, device=device)
        self.head = nn.Linear(dim, num_classes, dtype=dtype, device=device)

    def forward_features(self, x):
        x = self.patch_embed(x)
        for lvl, level in enumerate(self.levels):
            x = level(x)
            if lvl < len(self.downsamplers):
                x = self.downsamplers[lvl](x)
        return self.norm(x).mean(dim=(1, 2))

    def forward(self, x):
        return self.head(self.forward_features(x))


def nat_macs(variant: str = "tiny", res: tuple[int, int] = (224, 224), kernel_size: int = 7,
             num_classes: int = 1000) -> dict:
    """Analytic multiply-accumulate count of one image's forward, split by kind (the FLOPs column
    of Table 2 counts MACs).  NA: Q.K and P.V over min(k,H) x min(k,W) keys per query-head
    (Table 1's O(HW C L^2) term per level)."""
    cfg = VARIANTS[variant]
    heads = cfg["heads"]
    dim = heads * HEAD_DIM
    H, W = res

    def conv_out(n):
        return (n + 2 - 3) // 2 + 1

    macs = dict(conv=0, linear=0, na=0)
    h1, w1 = conv_out(H), conv_out(W)
    macs["conv"] += h1 * w1 * 9 * 3 * (dim // 2)
    H, W = conv_out(h1), conv_out(w1)
    macs["conv"] += H * W * 9 * (dim // 2) * dim
    for lvl, depth in enumerate(cfg["depths"]):
        hidden = int(math.ceil(dim * cfg["mlp_ratio"]))
        n = H * W
        per_block_lin = n * (dim * 3 * dim + dim * dim + 2 * dim * hidden)
        per_block_na = 2 * n * dim * min(kernel_size, H) * min(kernel_size, W)
        macs["linear"] += depth * per_block_lin
        macs["na"] += depth * per_block_na
        if lvl < len(cfg["depths"]) - 1:
            H, W = conv_out(H), conv_out(W)
            macs["conv"] += H * W * 9 * dim * 2 * dim
            dim *= 2
    macs["linear"] += dim * num_classes
    macs["total"] = macs["conv"] + macs["linear"] + macs["na"]
    return macs
