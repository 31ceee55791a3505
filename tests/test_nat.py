"""NAT model around the NA2D kernels.

CPU: the architecture reading (paper_2204_07143_b200/nat.py) is pinned to Table 2:
parameter counts 20/28/51/90 M and 2.7/4.3/7.8/13.7 GFLOPs at 224x224, both as printed (rounded).
GPU: a NAT-Mini forward in fp32 with every NA step through libna2d.so matches the same weights
with NA replaced by the dense masked-attention reference (tests/test_mhna.py); a NAT-Tiny
224x224 bf16 forward + backward runs on the tcgen05 kernels with finite logits and gradients.
"""
import pytest
import torch

from paper_2204_07143_b200.nat import NAT, VARIANTS, nat_macs

# Table 2: # Params (M), FLOPs (G)
TABLE2 = {"mini": (20, 2.7), "tiny": (28, 4.3), "small": (51, 7.8), "base": (90, 13.7)}


@pytest.mark.parametrize("variant", sorted(TABLE2))
def test_params_and_flops_match_table2(variant):
    params_m, gflops = TABLE2[variant]
    m = NAT(variant, device="meta")
    n = sum(p.numel() for p in m.parameters())
    assert round(n / 1e6) == params_m
    assert round(nat_macs(variant)["total"] / 1e9, 1) == gflops


def test_level_shapes():
    """Dims and heads double after every level (Table 2 caption); head dim 32; 3 downsamplers."""
    m = NAT("tiny", device="meta")
    dims = [lvl[0].attn.dim for lvl in m.levels]
    heads = [lvl[0].attn.heads for lvl in m.levels]
    assert dims == [64, 128, 256, 512] and heads == [2, 4, 8, 16]
    assert [len(lvl) for lvl in m.levels] == list(VARIANTS["tiny"]["depths"])
    assert len(m.downsamplers) == 3 and all(lvl[0].attn.head_dim == 32 for lvl in m.levels)
    # NA MACs: level maps 56, 28, 14, 7 at 224 (the last level's 7x7 window is the whole map)
    macs = nat_macs("tiny")
    na = 2 * (3 * 56 * 56 * 64 * 49 + 4 * 28 * 28 * 128 * 49 + 18 * 14 * 14 * 256 * 49 + 5 * 7 * 7 * 512 * 49)
    assert macs["na"] == na


@pytest.mark.gpu
def test_nat_mini_fp32_vs_dense_reference(monkeypatch):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2204_07143_b200.mhna as mhna
    from tests.test_mhna import dense_na_reference
    torch.manual_seed(0)
    model = NAT("mini", device="cuda", dtype=torch.float32).eval()
    with torch.no_grad():
        for mod in model.modules():
            if isinstance(mod, mhna.NeighborhoodAttention2D):
                mod.rpb.normal_()
    x = torch.randn(2, 3, 64, 64, device="cuda")  # level maps 16, 8, 4, 2 (k=7 >= map from level 2 on)
    with torch.no_grad():
        got = model(x)
        monkeypatch.setattr(mhna, "na2d", lambda q, k, v, rpb, kernel_size, scale: dense_na_reference(
            q, k, v, rpb, kernel_size, scale))
        ref = model(x)
    tol = 1e-4 * max(1.0, float(ref.abs().max()))
    assert float((got - ref).abs().max()) <= tol


@pytest.mark.gpu
def test_nat_tiny_224_bf16_fwd_bwd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.manual_seed(1)
    model = NAT("tiny", device="cuda")
    x = torch.randn(2, 3, 224, 224, device="cuda", dtype=torch.bfloat16)
    logits = model(x)
    assert logits.shape == (2, 1000) and torch.isfinite(logits).all()
    logits.float().logsumexp(-1).mean().backward()
    for name, p in model.named_parameters():
        assert p.grad is not None and torch.isfinite(p.grad).all(), name
    assert any(float(lvl[0].attn.rpb.grad.abs().sum()) > 0 for lvl in model.levels)
