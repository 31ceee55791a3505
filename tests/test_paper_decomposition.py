"""The paper's unfused NA decomposition: QK+RPB kernel writing
the attention weights, softmax, AV, and their gradients -- checked element by element against the
fp64 oracle with the north-star tolerances, and its attention weights against Eq. 2 directly."""
import numpy as np
import pytest

from na2d_inputs import Shape, make_inputs
from tests.parity import compare, run_oracle

pytestmark = pytest.mark.gpu

SHAPES = [Shape("p8x8k3", 1, 1, 8, 8, 32, 3), Shape("p13x18k7", 2, 2, 13, 18, 32, 7),
          Shape("p5x9k7", 1, 2, 5, 9, 32, 7), Shape("p11x10k5d64", 1, 2, 11, 10, 64, 5)]


@pytest.fixture(scope="module", autouse=True)
def cuda_lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s.name)
@pytest.mark.parametrize("dtype", ["bf16", "f32", "f16"])
def test_paper_path_vs_oracle(shape, dtype):
    import torch
    import paper_2204_07143_b200 as na2d
    inp = make_inputs(shape, seed=21, dtype=dtype)
    scale = shape.d ** -0.5
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dtype]
    t = {n: torch.from_numpy(inp[n]).cuda().to(tdt) for n in ("q", "k", "v", "dout")}
    rpb = torch.from_numpy(inp["rpb"]).cuda()
    out, lse, attn = na2d.paper_forward(t["q"], t["k"], t["v"], rpb, shape.kernel_size, scale)
    dq, dk, dv, drpb = na2d.paper_backward(t["q"], t["k"], t["v"], rpb, attn, t["dout"], shape.kernel_size, scale)
    torch.cuda.synchronize()
    got = {n: x.float().cpu().numpy() for n, x in dict(out=out, lse=lse, dq=dq, dk=dk, dv=dv, drpb=drpb).items()}
    ref = run_oracle(inp, shape.kernel_size, scale)
    compare(got, ref, dtype)
    a = attn.cpu().numpy()
    np.testing.assert_allclose(a.sum(-1), 1.0, atol=1e-5)  # every row is a distribution over its window
    assert a.shape[-1] == min(shape.kernel_size, shape.H) * min(shape.kernel_size, shape.W)


def test_paper_path_matches_fused_path():
    """Same inputs through the fused tcgen05 kernels and the paper's decomposition (bf16)."""
    import torch
    import paper_2204_07143_b200 as na2d
    s = Shape("cmp", 2, 2, 24, 33, 32, 7)
    inp = make_inputs(s, seed=4)
    t = {n: torch.from_numpy(inp[n]).cuda().bfloat16() for n in ("q", "k", "v", "dout")}
    rpb = torch.from_numpy(inp["rpb"]).cuda()
    o1, l1 = na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
    o2, l2, _ = na2d.paper_forward(t["q"], t["k"], t["v"], rpb, 7)
    torch.cuda.synchronize()
    assert float((o1.float() - o2.float()).abs().max()) <= 2e-2
    assert float((l1 - l2).abs().max()) <= 1e-3
