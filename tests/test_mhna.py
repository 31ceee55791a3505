"""MHNA layer: autograd over the NA2D C ABI, checked against the fp64 oracle
(gradients of Eq. 2) and against an independent dense masked-attention layer written here in
plain torch (fp32), with the same weights."""
import numpy as np
import pytest
import torch

from na2d_inputs import Shape, make_inputs


def test_layer_construction_cpu():
    """Host-side: parameter shapes and the Eq. 2 bias convention (R1), no CUDA calls."""
    from paper_2204_07143_b200.mhna import NeighborhoodAttention2D
    m = NeighborhoodAttention2D(64, 2, 7, dtype=torch.float32)
    assert m.rpb.shape == (2, 13, 13)
    assert m.qkv.weight.shape == (192, 64) and m.proj.weight.shape == (64, 64)
    # trunc-normal(0, 0.02) table (Swin / timm: truncated at +-2 absolute) divided by
    # scale = 32**-0.5 (B = B_swin / scale): std 0.02 * sqrt(32)
    tbl = m.rpb.detach()
    assert abs(float(tbl.std()) - 0.02 * 32 ** 0.5) < 0.02 and float(tbl.abs().max()) < 10 * 0.02 * 32 ** 0.5
    with pytest.raises(ValueError):
        NeighborhoodAttention2D(64, 3, 7)
    with pytest.raises(ValueError):
        NeighborhoodAttention2D(64, 2, 4)


def _window_start(i, n, L):
    if L >= n:
        return 0
    return min(max(i - (L - 1) // 2, 0), n - L)


def dense_na_reference(q, k, v, rpb, L, scale):
    """Eq. 2 as dense attention over the H*W keys with a -inf mask outside each query's clamped
    window and the bias B[h, p-i+L-1, q-j+L-1] added inside it (fp32, plain torch)."""
    B, heads, H, W, d = q.shape
    n = H * W
    mask = torch.full((n, n), float("-inf"), device=q.device)
    bias = torch.zeros((heads, n, n), device=q.device)
    for i in range(H):
        si = _window_start(i, H, L)
        for j in range(W):
            sj = _window_start(j, W, L)
            for p in range(si, si + min(L, H)):
                for qq in range(sj, sj + min(L, W)):
                    mask[i * W + j, p * W + qq] = 0.0
                    if rpb is not None:
                        bias[:, i * W + j, p * W + qq] = rpb[:, p - i + L - 1, qq - j + L - 1]
    qf, kf, vf = (t.reshape(B, heads, n, d) for t in (q, k, v))
    s = scale * (qf @ kf.transpose(-1, -2) + bias) + mask
    return (torch.softmax(s, -1) @ vf).reshape(B, heads, H, W, d)


class DenseMHNA(torch.nn.Module):
    """The layer of paper_2204_07143_b200.mhna with the dense reference in place of the kernels."""

    def __init__(self, m):
        super().__init__()
        self.m = m

    def forward(self, x):
        m = self.m
        b, h, w, c = x.shape
        qkv = m.qkv(x).view(b, h, w, 3, m.heads, m.head_dim).permute(3, 0, 4, 1, 2, 5)
        o = dense_na_reference(qkv[0], qkv[1], qkv[2], m.rpb, m.kernel_size, m.scale)
        return m.proj(o.permute(0, 2, 3, 1, 4).reshape(b, h, w, c))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_na2d_function_grads_vs_oracle(dtype):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    from paper_2204_07143_b200.mhna import na2d
    from tests.parity import compare
    s = Shape("fn", 2, 2, 13, 18, 32, 7)
    inp = make_inputs(s, seed=5, dtype=dtype)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    t = {n: torch.from_numpy(inp[n]).cuda().to(tdt).requires_grad_(n != "dout") for n in ("q", "k", "v", "dout")}
    rpb = torch.from_numpy(inp["rpb"]).cuda().requires_grad_(True)
    out = na2d(t["q"], t["k"], t["v"], rpb, 7)
    out.backward(t["dout"])
    ref = oracle.na2d_backward(inp["q"], inp["k"], inp["v"], inp["rpb"], inp["dout"], 7, 32 ** -0.5)
    got = dict(out=out.detach().float().cpu().numpy(), dq=t["q"].grad.float().cpu().numpy(),
               dk=t["k"].grad.float().cpu().numpy(), dv=t["v"].grad.float().cpu().numpy(),
               drpb=rpb.grad.cpu().numpy())
    compare(got, ref, dtype, names=["out", "dq", "dk", "dv", "drpb"])


@pytest.mark.gpu
def test_mhna_layer_vs_dense_reference():
    """Layer output and every parameter gradient vs the dense masked-attention layer (fp32 path,
    1e-4 relative: the reference and the kernels both compute in fp32)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_07143_b200.mhna import NeighborhoodAttention2D
    torch.manual_seed(0)
    m = NeighborhoodAttention2D(64, 2, 5, dtype=torch.float32, device="cuda")
    with torch.no_grad():
        m.rpb.normal_()
    ref = DenseMHNA(m)
    x = torch.randn(2, 9, 11, 64, device="cuda", requires_grad=True)
    g = torch.randn(2, 9, 11, 64, device="cuda")
    y = m(x)
    grads = torch.autograd.grad(y, [x] + list(m.parameters()), g)
    y_ref = ref(x)
    grads_ref = torch.autograd.grad(y_ref, [x] + list(m.parameters()), g)
    np.testing.assert_allclose(y.detach().cpu().numpy(), y_ref.detach().cpu().numpy(), rtol=1e-4, atol=1e-4)
    for a, b in zip(grads, grads_ref):
        tol = 1e-4 * max(1.0, float(b.abs().max()))
        assert float((a - b).abs().max()) <= tol


@pytest.mark.gpu
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16], ids=["bf16", "f16"])
def test_nat_block_stage1_step(dt):
    """One NAT-Tiny stage-1 block (C=64, 2 heads, k=7, 56x56) forward + backward in bf16 / fp16 on
    the tcgen05 kernels: finite outputs and gradients reaching every parameter."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_07143_b200.mhna import NATBlock
    torch.manual_seed(1)
    blk = NATBlock(64, 2, 7, device="cuda", dtype=dt)
    x = torch.randn(4, 56, 56, 64, device="cuda", dtype=dt, requires_grad=True)
    y = blk(x)
    y.float().square().mean().backward()
    assert torch.isfinite(y).all()
    for p in list(blk.parameters()) + [x]:
        assert p.grad is not None and torch.isfinite(p.grad).all()
    assert blk.attn.rpb.grad.abs().sum() > 0
