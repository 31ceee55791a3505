"""GPU parity (-m gpu): the CUDA path through the C ABI vs the fp64 oracle on the same seeded
inputs, element by element, with the north-star tolerances (tests/parity.py).  Covers the
BASELINE configs at full size (the launch configuration bench.py times), ragged tiles, L >= map
size, single-pixel maps, no-RPB, row bands, both kernel families and RPB probes."""
import os

import numpy as np
import pytest

from na2d_inputs import CONFIGS, Shape, make_inputs
from tests.parity import compare, log_errors, run_cuda, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def cuda_lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_07143_b200 import build
    build.build()


def check(shape: Shape, dtype="bf16", rpb="parity", seed=None, backward=True, **band):
    inp = make_inputs(shape, seed=seed, dtype=dtype, rpb=rpb)
    scale = shape.d ** -0.5
    ref = run_oracle(inp, shape.kernel_size, scale, backward=backward)
    got = run_cuda(inp, shape.kernel_size, scale, dtype, backward=backward)
    rep = compare(got, ref, dtype)
    log_errors(shape.name, dtype, rep)
    return rep


def family(shape: Shape, dtype="bf16"):
    import paper_2204_07143_b200 as na2d
    code = {"bf16": na2d.NA2D_BF16, "f16": na2d.NA2D_F16, "f32": na2d.NA2D_F32}[dtype]
    p = na2d.make_problem(shape.B, shape.heads, shape.H, shape.W, shape.d, shape.kernel_size, code)
    return na2d.na2d_kernel_family(p, 0), na2d.na2d_kernel_family(p, 1)


SMALL = [
    Shape("s8x8k3", 1, 1, 8, 8, 32, 3),          # BASELINE config 1
    Shape("ragged13x29k7", 2, 2, 13, 29, 32, 7),  # ragged in both axes
    Shape("ragged30x17k5", 1, 3, 30, 17, 32, 5),
    Shape("k_gt_map5x5k7", 2, 1, 5, 5, 32, 7),   # window covers the map
    Shape("k_gt_w9x4k7", 1, 2, 9, 4, 32, 7),     # L > W only
    Shape("pixel1x1k3", 3, 2, 1, 1, 32, 3),      # single pixel: O = V
    Shape("wide3x70k3", 1, 1, 3, 70, 32, 3),
    Shape("sa7x7k7", 4, 4, 7, 7, 32, 7),         # NAT-Tiny stage-4 geometry (k = map: full SA)
    Shape("tall61x9k7", 1, 1, 61, 9, 32, 7),
    Shape("w37k7", 2, 2, 11, 37, 32, 7),         # W = 5 mod 16: shifted key tile columns (B2)
    Shape("w54k7", 1, 2, 9, 54, 32, 7),          # W = 6 mod 16
]


@pytest.mark.parametrize("shape", SMALL, ids=lambda s: s.name)
@pytest.mark.parametrize("dtype", ["bf16", "f32", "f16"])
def test_small_shapes(shape, dtype):
    check(shape, dtype)


@pytest.mark.parametrize("dtype", ["bf16", "f32", "f16"])
def test_no_rpb(dtype):
    check(Shape("norpb", 2, 2, 19, 23, 32, 7), dtype, rpb=None)


@pytest.mark.parametrize("d,L", [(16, 3), (64, 5), (128, 3), (32, 9), (32, 11), (8, 13)])
@pytest.mark.parametrize("dtype", ["bf16", "f32", "f16"])
def test_other_dims_and_kernel_sizes(d, L, dtype):
    check(Shape(f"d{d}k{L}", 2, 2, 17, 21, d, L), dtype)


TC_DIMS = [Shape(f"tc_d{d}_{n}", *dims[:4], d, dims[4]) for d in (16, 64)
           for n, dims in (("ragged13x29k7", (2, 2, 13, 29, 7)), ("ragged30x17k5", (1, 3, 30, 17, 5)),
                           ("17x21k3", (2, 2, 17, 21, 3)), ("sa7x7k7", (3, 2, 7, 7, 7)), ("w37k7", (1, 2, 11, 37, 7)))]


@pytest.mark.parametrize("shape", TC_DIMS, ids=lambda s: s.name)
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_tensor_core_forward_other_head_dims(shape, dtype):
    """f3: head dims 16 and 64 run the tcgen05 forward and backward (32 / 128-byte
    swizzled operand rows); every output element by element."""
    fam = family(shape, dtype)
    assert fam == ("tcgen05", "tcgen05"), fam
    check(shape, dtype)


@pytest.mark.parametrize("d", [16, 64])
def test_tensor_core_forward_other_head_dims_full_size(d):
    """NAT-Tiny stage-1 geometry with head dim d (B = 16): the tcgen05 kernels at size, forward and
    backward, element by element against the oracle."""
    shape = Shape(f"tc_d{d}_s1", 16, 2, 56, 56, d, 7)
    assert family(shape) == ("tcgen05", "tcgen05")
    check(shape)


@pytest.mark.parametrize("L", [3, 5, 7])
def test_rpb_one_hot_probe(L):
    """Q = 0, one large table cell: every query whose window holds that offset copies V there.
    Pins bias sign/orientation incl. the corner cells (1 (query,key) pair per map)."""
    import torch
    import paper_2204_07143_b200 as na2d
    H, W, d = 20, 37, 32
    T = 2 * L - 1
    g = np.random.default_rng(L)
    from na2d_inputs import bf16_round
    v = bf16_round(g.standard_normal((1, 1, H, W, d)).astype(np.float32))
    k = bf16_round(g.standard_normal((1, 1, H, W, d)).astype(np.float32))
    q = np.zeros_like(v)
    tq, tk, tv = (torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v))
    for a, c in [(0, 0), (T - 1, T - 1), (0, T - 1), (T - 1, 0), (L - 1, L - 1), (1, L + 1)]:
        rpb = np.zeros((1, T, T), np.float32)
        rpb[0, a, c] = 2000.0
        out, _ = na2d.forward(tq, tk, tv, torch.from_numpy(rpb).cuda(), L, 0.125)
        out = out.float().cpu().numpy()
        import oracle
        ref, _ = oracle.na2d_forward(q, k, v, rpb, L, 0.125)
        np.testing.assert_allclose(out, ref, atol=2e-2)
        hits = 0
        for i in range(H):
            for j in range(W):
                p, qq = i + a - (L - 1), j + c - (L - 1)
                si, sj = oracle.window_start(i, H, L), oracle.window_start(j, W, L)
                if si <= p < si + L and sj <= qq < sj + L:
                    hits += 1
                    np.testing.assert_allclose(out[0, 0, i, j], v[0, 0, p, qq], atol=1e-2)
        assert hits >= 1


@pytest.mark.parametrize("L", [3, 5, 7])
def test_drpb_cell_probe(L):
    """dRPB cell by cell (SURVEY c-11 peripheral cells): head h has dO = 0 except at one probe
    query, so dRPB[h] is nonzero only on that query's L x L window cells and a zeroed, moved or
    sign-flipped cell (the corner cells get a single term) fails.  The four corner queries hit
    the four corner cells of the table."""
    import torch
    import oracle
    import paper_2204_07143_b200 as na2d
    from na2d_inputs import bf16_round
    H, W, d = 20, 37, 32
    T = 2 * L - 1
    probes = [(0, 0), (0, W - 1), (H - 1, 0), (H - 1, W - 1), (H // 2, W // 2), (1, W - 2), (L // 2 + 1, 2)]
    heads = len(probes)
    g = np.random.default_rng(100 + L)
    q, k, v = (bf16_round(g.standard_normal((1, heads, H, W, d)).astype(np.float32)) for _ in range(3))
    dout = np.zeros_like(q)
    for h, (i, j) in enumerate(probes):
        dout[0, h, i, j] = bf16_round(g.standard_normal(d).astype(np.float32))
    rpb = (g.standard_normal((heads, T, T)) * np.sqrt(d)).astype(np.float32)
    scale = d ** -0.5
    ref = oracle.na2d_backward(q, k, v, rpb, dout, L, scale)
    tq, tk, tv, tdo = (torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v, dout))
    trpb = torch.from_numpy(rpb).cuda()
    out, lse = na2d.forward(tq, tk, tv, trpb, L, scale)
    drpb = na2d.backward(tq, tk, tv, trpb, out, lse, tdo, L, scale)[3].cpu().numpy()
    for h, (i, j) in enumerate(probes):
        si, sj = oracle.window_start(i, H, L), oracle.window_start(j, W, L)
        mask = np.zeros((T, T), bool)
        mask[si - i + L - 1:si - i + 2 * L - 1, sj - j + L - 1:sj - j + 2 * L - 1] = True
        assert np.all(drpb[h][~mask] == 0.0), f"probe {h}: cells outside the window written"
        assert np.all(ref["drpb"][h][~mask] == 0.0)
        np.testing.assert_allclose(drpb[h], ref["drpb"][h], rtol=1e-3, atol=1e-5, err_msg=f"probe {h} at {(i, j)}")
    corners = {(0, 0): (T - 1, T - 1), (0, W - 1): (T - 1, 0), (H - 1, 0): (0, T - 1), (H - 1, W - 1): (0, 0)}
    for h, (i, j) in enumerate(probes[:4]):
        a, c = corners[(i, j)]
        assert abs(ref["drpb"][h, a, c]) > 1e-4 and np.sign(drpb[h, a, c]) == np.sign(ref["drpb"][h, a, c])


@pytest.mark.parametrize("L", [3, 5, 7])
def test_large_bias_range(L):
    """A bias range of ~10^2 (log2 units) inside one window: the forward's upper-bound softmax shift
    (raw-S max + window bias max) underflows the row sum there, and its exact-max redo must give
    the oracle's result (forward and backward)."""
    shape = Shape(f"bigbias{L}", 2, 2, 19, 37, 32, L)
    inp = make_inputs(shape, seed=21 + L)
    # a near one-hot softmax passes |v| straight to O: V, dO halved (exact in bf16) keep |O| < 4, where
    # the bf16 output rounding alone stays below 2^-8 (the north-star inputs' regime)
    inp["v"], inp["dout"] = inp["v"] * 0.5, inp["dout"] * 0.5
    scale = shape.d ** -0.5
    base = inp["rpb"]
    for mul, bwd in [(25.0, False), (10.0, True)]:  # window bias ranges ~160 / ~65 (log2 units)
        inp["rpb"] = (base * mul).astype(np.float32)
        ref = run_oracle(inp, L, scale, backward=bwd)
        got = run_cuda(inp, L, scale, "bf16", backward=bwd)
        log_errors(f"{shape.name}x{mul:g}", "bf16", compare(got, ref, "bf16"))


@pytest.mark.parametrize("dtype,d", [("bf16", 32), ("f32", 32), ("f16", 32), ("bf16", 16), ("bf16", 64)])
def test_row_band(dtype, d):
    """Band call (global coordinates) == oracle band call, incl. dk/dv partials (d = 16 / 64: the
    head-dim variants of the tcgen05 kernels in band geometry)."""
    shape = Shape("band", 2, 2, 40, 27, d, 7)
    inp = make_inputs(shape, seed=77, dtype=dtype)
    import oracle
    for r0, r1 in [(0, 20), (20, 40), (13, 29)]:
        k0 = oracle.window_start(r0, 40, 7)
        k1 = oracle.window_start(r1 - 1, 40, 7) + 7
        sub = dict(q=inp["q"][:, :, r0:r1], k=inp["k"][:, :, k0:k1], v=inp["v"][:, :, k0:k1],
                   dout=inp["dout"][:, :, r0:r1], rpb=inp["rpb"])
        ref = run_oracle(sub, 7, d ** -0.5, H=40, q_row0=r0, kv_row0=k0)
        got = run_cuda(sub, 7, d ** -0.5, dtype, H=40, q_row0=r0, kv_row0=k0)
        compare(got, ref, dtype)


@pytest.mark.parametrize("name", list(CONFIGS), ids=str)
def test_baseline_configs_full_size(name):
    """Every BASELINE.json config at full size, fwd + bwd, all outputs element by element
    (the oracle runs on all host cores)."""
    # north_star "no other paths": every BASELINE config must run on the tcgen05 kernels
    assert family(CONFIGS[name]) == ("tcgen05", "tcgen05"), family(CONFIGS[name])
    rep = check(CONFIGS[name], "bf16")
    print(name, {k: f"{e:.2e}/{t:.1e}" for k, (e, t) in rep.items()})


def test_config1_fp32():
    check(CONFIGS["cfg1_8x8_k3"], "f32")


def test_config2_fp16_full_size():
    """fp16 I/O (NA2D_F16) on the same tcgen05 kernels at the stage-1 configuration."""
    assert family(CONFIGS["cfg2_nat_tiny_s1"], "f16") == ("tcgen05", "tcgen05")
    rep = check(CONFIGS["cfg2_nat_tiny_s1"], "f16")
    print("cfg2 f16", {k: f"{e:.2e}/{t:.1e}" for k, (e, t) in rep.items()})


def test_kernel_family_and_launches():
    import paper_2204_07143_b200 as na2d
    s = CONFIGS["cfg2_nat_tiny_s1"]
    p = na2d.make_problem(s.B, s.heads, s.H, s.W, s.d, s.kernel_size)
    fam = (na2d.na2d_kernel_family(p, 0), na2d.na2d_kernel_family(p, 1))
    print("cfg2 kernel families", fam)
    assert na2d.na2d_launch_count(p, 0) >= 1 and na2d.na2d_launch_count(p, 1) >= 1


def test_step_host_matches_device_path():
    """The host-buffer end-to-end entry point gives the device path's results."""
    import ctypes
    import torch
    import paper_2204_07143_b200 as na2d
    s = Shape("host", 2, 2, 21, 18, 32, 7)
    inp = make_inputs(s, seed=3)
    ref = run_cuda(inp, 7, 32 ** -0.5, "bf16")
    p = na2d.make_problem(s.B, s.heads, s.H, s.W, s.d, 7)
    host = {n: torch.from_numpy(inp[n]).bfloat16().pin_memory() for n in ("q", "k", "v", "dout")}
    rpb = torch.from_numpy(inp["rpb"]).pin_memory()
    outs = {n: torch.empty_like(host["q"]).pin_memory() for n in ("out", "dq", "dk", "dv")}
    lse = torch.empty(host["q"].shape[:4]).pin_memory()
    drpb = torch.empty_like(rpb).pin_memory()
    nbytes = na2d.na2d_step_host_workspace_bytes(p)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    na2d.na2d_step_host(p, host["q"].data_ptr(), host["k"].data_ptr(), host["v"].data_ptr(), rpb.data_ptr(),
                        host["dout"].data_ptr(), outs["out"].data_ptr(), lse.data_ptr(), outs["dq"].data_ptr(),
                        outs["dk"].data_ptr(), outs["dv"].data_ptr(), drpb.data_ptr(), ws.data_ptr(), nbytes, st)
    torch.cuda.synchronize()
    for n in ("out", "dq", "dk", "dv"):
        np.testing.assert_array_equal(outs[n].float().numpy(), ref[n])
    np.testing.assert_allclose(lse.numpy(), ref["lse"], atol=1e-6)
    np.testing.assert_allclose(drpb.numpy(), ref["drpb"], atol=1e-3, rtol=1e-4)


@pytest.mark.parametrize("shape,dtype", [
    (Shape("nan7", 2, 2, 19, 37, 32, 7), "bf16"),   # ragged tiles, B2 shifted key columns (W = 5 mod 16)
    (Shape("nan5", 1, 2, 13, 21, 32, 5), "bf16"),
    (Shape("nan3", 1, 1, 9, 18, 32, 3), "bf16"),
    (Shape("nanf", 1, 2, 11, 14, 32, 7), "f32"),
], ids=lambda x: x.name if isinstance(x, Shape) else x)
def test_every_output_element_written(shape, dtype):
    """Outputs pre-filled with NaN come back fully overwritten (out, lse, dq, dk, dv, drpb) and
    equal to the oracle.  compute-sanitizer's initcheck does not see the TMA (bulk async) stores
    of the tensor-core kernels, so this is the direct check that every element is written."""
    import torch
    import oracle
    import paper_2204_07143_b200 as na2d
    from tests.parity import compare
    inp = make_inputs(shape, seed=9, dtype=dtype)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    t = {n: torch.from_numpy(inp[n]).cuda().to(tdt) for n in ("q", "k", "v", "dout")}
    rpb = torch.from_numpy(inp["rpb"]).cuda()
    nan = lambda like, dt=None: torch.full_like(like, float("nan"), dtype=dt or like.dtype)  # noqa: E731
    out, lse = nan(t["q"]), torch.full(t["q"].shape[:4], float("nan"), device="cuda")
    na2d.forward(t["q"], t["k"], t["v"], rpb, shape.kernel_size, out=out, lse=lse)
    grads = (nan(t["q"]), nan(t["k"]), nan(t["v"]), nan(rpb))
    na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], shape.kernel_size, grads=grads)
    torch.cuda.synchronize()
    got = dict(out=out, lse=lse, dq=grads[0], dk=grads[1], dv=grads[2], drpb=grads[3])
    for n, x in got.items():
        assert not torch.isnan(x).any(), f"{n}: {int(torch.isnan(x).sum())} elements never written"
    ref = oracle.na2d_backward(inp["q"], inp["k"], inp["v"], inp["rpb"], inp["dout"], shape.kernel_size,
                               shape.d ** -0.5)
    compare({n: x.float().cpu().numpy() for n, x in got.items()}, ref, dtype,
            names=["out", "lse", "dq", "dk", "dv", "drpb"])


@pytest.mark.parametrize("dtype,d", [("f32", 32), ("bf16", 32), ("bf16", 128)])
def test_drpb_bitwise_reproducible(dtype, d):
    """dRPB is summed in a fixed order on both paths (tcgen05: per-CTA tables reduced in CTA order;
    SIMT: per-query window-slot dS reduced per cell in a fixed order): two runs give identical bits."""
    import torch
    import paper_2204_07143_b200 as na2d
    shape = Shape(f"det_{dtype}_d{d}", 2, 2, 19, 23, d, 7)
    inp = make_inputs(shape, seed=5, dtype=dtype)
    el = {"f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    t = {n: torch.from_numpy(inp[n]).cuda().to(el) for n in ("q", "k", "v", "dout")}
    rpb = torch.from_numpy(inp["rpb"]).cuda()
    out, lse = na2d.forward(t["q"], t["k"], t["v"], rpb, 7)
    a = na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)[3].clone()
    b = na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], 7)[3].clone()
    assert torch.equal(a, b)


# Small-map pair mode (tc::pair_mode: H, W <= 8, even B, whole map): two maps per 8 x 16 tile,
# each with its own clamped windows and bias cells.  Shapes cover W <= 4 (quarters 1 and 3 empty),
# L > map, L < map (clamped windows inside each member), odd and even widths.
PAIR = [
    Shape("pair7x7k7", 4, 3, 7, 7, 32, 7),     # NAT-Tiny stage 4 geometry
    Shape("pair8x8k3", 2, 2, 8, 8, 32, 3),
    Shape("pair6x8k5", 6, 1, 6, 8, 32, 5),
    Shape("pair8x5k7", 2, 2, 8, 5, 32, 7),
    Shape("pair3x4k3", 4, 2, 3, 4, 32, 3),
    Shape("pair7x7k5", 2, 2, 7, 7, 32, 5),
    Shape("pair2x7k3", 8, 1, 2, 7, 32, 3),
]


@pytest.mark.parametrize("shape", PAIR, ids=lambda s: s.name)
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_pair_mode_small_maps(shape, dtype):
    assert family(shape, dtype) == ("tcgen05", "tcgen05")
    check(shape, dtype)


@pytest.mark.parametrize("d", [16, 64])
@pytest.mark.parametrize("L", [3, 7])
def test_pair_mode_head_dims(d, L):
    check(Shape(f"pair7x6d{d}k{L}", 4, 2, 7, 6, d, L), "bf16")


def test_pair_mode_outputs_all_written():
    test_every_output_element_written(Shape("nanpair", 4, 2, 7, 7, 32, 7), "bf16")


@pytest.mark.parametrize("rpb", [None, "parity"])
def test_pair_mode_many_heads_no_bias(rpb):
    """Pair mode with more than 64 heads (B1's per-CTA committed-heads mask falls back to
    read-modify-write of the partial tables) and with no RPB at all."""
    check(Shape("pair70h", 2, 70, 8, 8, 32, 3), "bf16", rpb=rpb)


def test_many_heads_class_switches():
    """More than 64 heads on a multi-tile map: B1 CTAs cross (class, head) segments and commit
    heads >= 64 by read-modify-write.  (This input reaches |dV| = 4.5: bound R7b applies there.)"""
    check(Shape("h72", 1, 72, 20, 20, 32, 5), "bf16")


FUZZ = []
_rng = np.random.default_rng(20441)
for _n in range(24):
    _L = int(_rng.choice([3, 5, 7]))
    _H, _W = int(_rng.integers(1, 41)), int(_rng.integers(1, 41))
    _B = int(_rng.choice([1, 2, 3, 4, 6]))
    _heads = int(_rng.integers(1, 5))
    _d = int(_rng.choice([16, 32, 64]))
    FUZZ.append((Shape(f"fuzz{_n}_{_B}x{_heads}x{_H}x{_W}d{_d}k{_L}", _B, _heads, _H, _W, _d, _L),
                 "f16" if _n % 3 == 2 else "bf16"))


@pytest.mark.parametrize("shape,dtype", FUZZ, ids=lambda x: x.name if isinstance(x, Shape) else x)
def test_fuzz_shapes(shape, dtype):
    """Seeded random geometry (maps 1..40 per axis incl. pair-mode sizes, batch / heads, d, L, bf16 /
    fp16) against the oracle: catches tile-order, range-balancing, pair-mode and border-path slips."""
    check(shape, dtype)
