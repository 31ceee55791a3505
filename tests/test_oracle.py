"""Pins for the fp64 oracle (-m "not gpu").  Each test checks the oracle against something
other than itself: printed worked examples (tests/golden/), independent formulations
(brute-force argmin window, Appendix A unfold + replicate pad, Eq. 1 dense attention with
an enumerated mask, torch.autograd), closed forms, invariants and finite differences.
Citations: P:<line> = PAPER.md, S:<line> = SPEC.md."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import reference as ref
from na2d_inputs import Shape, make_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "geometry_examples.json")


def rnd(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


def rand_problem(B, heads, H, W, d, L, seed, bias_scale=1.0, with_bias=True):
    g = np.random.default_rng(seed)
    q, k, v, do = (g.standard_normal((B, heads, H, W, d)) for _ in range(4))
    T = 2 * L - 1
    rpb = g.standard_normal((heads, T, T)) * bias_scale * np.sqrt(d) if with_bias else None
    return q, k, v, do, rpb


# ---------------------------------------------------------------- geometry (a1, a2)

def test_golden_geometry_examples(oracle_lib):
    gold = json.load(open(GOLDEN))
    for ex in gold["window_start"]:
        assert oracle.window_start(ex["i"], ex["n"], ex["L"]) == ex["start"], ex
        assert oracle.window_len(ex["n"], ex["L"]) == ex["len"], ex
    for ex in gold["neighborhood"]:
        si = oracle.window_start(ex["i"], ex["H"], ex["L"])
        sj = oracle.window_start(ex["j"], ex["W"], ex["L"])
        rows = list(range(si, si + oracle.window_len(ex["H"], ex["L"])))
        cols = list(range(sj, sj + oracle.window_len(ex["W"], ex["L"])))
        assert rows == ex["rows"] and cols == ex["cols"], ex
    for ex in gold["rel_index"]:
        assert oracle.rel_index(ex["i"], ex["p"], ex["L"]) == ex["index"], ex


@pytest.mark.parametrize("L", [3, 5, 7, 9, 11, 13])
def test_window_three_formulations_agree(oracle_lib, L):
    """clamp (oracle) == nearest-centre argmin == unfold+replicate pad."""
    for n in range(1, 41):
        rows = np.arange(n, dtype=np.float64)[:, None, None] * np.ones((1, 1, 1))
        win = ref.unfold_windows(rows, L)[:, 0, :, 0, 0]  # [n, Lh] key rows per query
        for i in range(n):
            s = oracle.window_start(i, n, L)
            ln = oracle.window_len(n, L)
            assert s == ref.window_start_argmin(i, n, L)
            assert list(win[i].astype(int)) == list(range(s, s + ln))
            assert s <= i < s + ln                      # query inside own window
            assert 0 <= s and s + ln <= n
            if i:
                assert s >= oracle.window_start(i - 1, n, L)  # monotone
            if n >= L:
                assert ln == L                          # |rho| = L^2 incl. corners
                if (L - 1) // 2 <= i < n - (L - 1) // 2:
                    assert s == i - (L - 1) // 2        # interior queries centred


@pytest.mark.parametrize("L", [3, 5, 7])
def test_rel_index_range_centre_and_reflection(oracle_lib, L):
    for n in range(L, 30):
        seen = set()
        for i in range(n):
            s = oracle.window_start(i, n, L)
            assert oracle.rel_index(i, i, L) == L - 1   # self offset hits the centre cell
            # reflection: start(n-1-i) = (n-L) - start(i)  =>  idx(refl) = 2(L-1) - idx
            assert oracle.window_start(n - 1 - i, n, L) == (n - L) - s
            for p in range(s, s + L):
                idx = oracle.rel_index(i, p, L)
                seen.add(idx)
                assert oracle.rel_index(n - 1 - i, n - 1 - p, L) == 2 * (L - 1) - idx
        assert seen == set(range(2 * L - 1))            # range exactly [0, 2L-2]


@pytest.mark.parametrize("L", [3, 5, 7])
def test_inverse_neighbourhood_counts(oracle_lib, L):
    """Per axis each key is seen by NS+1 .. 3NS+1 queries once n >= 2L (shorter axes let the
    two clamped border windows overlap the middle), and the counts always sum to n*L."""
    ns = (L - 1) // 2
    for n in range(L, 40):
        cnt = np.zeros(n, int)
        for i in range(n):
            s = oracle.window_start(i, n, L)
            cnt[s:s + L] += 1
        assert cnt.sum() == n * L
        assert cnt.min() >= ns + 1
        if n >= 2 * L:
            assert cnt.max() <= 3 * ns + 1


# ---------------------------------------------------------------- forward (a3-a5)

@pytest.mark.parametrize("heads,L", [(1, 5), (2, 5), (1, 7), (2, 7)])
def test_na_equals_self_attention_when_window_covers_map(oracle_lib, heads, L):
    """P:141 / P:158: L >= feature-map size and no bias => NA == Eq. 1."""
    q, k, v, _, _ = rand_problem(1, heads, 5, 5, 8, L, seed=10 + L + heads, with_bias=False)
    out, _ = oracle.na2d_forward(q, k, v, None, L, 8 ** -0.5)
    for h in range(heads):
        sa = ref.self_attention(q[0, h].reshape(25, 8), k[0, h].reshape(25, 8), v[0, h].reshape(25, 8))
        np.testing.assert_allclose(out[0, h].reshape(25, 8), sa, atol=1e-12, rtol=0)


@pytest.mark.parametrize("L", [3, 5, 7])
def test_forward_matches_unfold_reference_grid(oracle_lib, L):
    """Appendix A unfold+replicate-pad formulation over H,W in 3..12."""
    seed = 0
    for H in range(3, 13, 2):
        for W in range(3, 13, 3):
            for heads, d in ((1, 2), (2, 4), (1, 8)):
                seed += 1
                q, k, v, _, rpb = rand_problem(1, heads, H, W, d, L, seed)
                out, lse = oracle.na2d_forward(q, k, v, rpb, L, d ** -0.5)
                o2, l2 = ref.na2d_unfold_forward(q, k, v, rpb, L, d ** -0.5)
                np.testing.assert_allclose(out, o2, atol=1e-12, rtol=0)
                np.testing.assert_allclose(lse, l2, atol=1e-12, rtol=0)


@pytest.mark.parametrize("H,W,L", [(8, 8, 3), (6, 9, 5), (9, 7, 7), (4, 11, 5), (3, 3, 7)])
def test_forward_matches_dense_masked_attention(oracle_lib, H, W, L):
    import torch
    q, k, v, _, rpb = rand_problem(2, 2, H, W, 8, L, seed=H * 100 + W * 10 + L)
    out, lse = oracle.na2d_forward(q, k, v, rpb, L, 8 ** -0.5)
    t = [torch.from_numpy(x) for x in (q, k, v, rpb)]
    o2, l2 = ref.na2d_dense(t[0], t[1], t[2], t[3], L, 8 ** -0.5)
    np.testing.assert_allclose(out, o2.numpy(), atol=1e-12, rtol=0)
    np.testing.assert_allclose(lse, l2.numpy(), atol=1e-12, rtol=0)


def test_special_cases(oracle_lib):
    # H=W=1 -> O = V
    q, k, v, _, rpb = rand_problem(2, 2, 1, 1, 4, 3, seed=1)
    out, lse = oracle.na2d_forward(q, k, v, rpb, 3)
    np.testing.assert_allclose(out, v, atol=1e-15)
    # LSE of a single logit = the logit itself = scale*(q.k + centre bias)
    np.testing.assert_allclose(lse[..., 0, 0], 0.5 * ((q * k).sum(-1)[..., 0, 0] + rpb[:, 2, 2][None]), atol=1e-12)
    # all K equal and no bias -> window mean of V
    H, W, L = 9, 10, 5
    q, _, v, _, _ = rand_problem(1, 1, H, W, 4, L, seed=2)
    k = np.broadcast_to(rnd((1, 1, 1, 1, 4), 3), q.shape).copy()
    out, _ = oracle.na2d_forward(q, k, v, None, L)
    for i in range(H):
        for j in range(W):
            si, sj = ref.window_start_argmin(i, H, L), ref.window_start_argmin(j, W, L)
            np.testing.assert_allclose(out[0, 0, i, j], v[0, 0, si:si + L, sj:sj + L].mean((0, 1)), atol=1e-12)
    # constant V -> O = that constant, whatever Q, K, bias
    q, k, _, _, rpb = rand_problem(1, 2, 7, 6, 4, 3, seed=4)
    v = np.full(q.shape, 0.375)
    out, _ = oracle.na2d_forward(q, k, v, rpb, 3)
    np.testing.assert_allclose(out, 0.375, atol=1e-14)


@pytest.mark.parametrize("L", [3, 5, 7])
def test_rpb_one_hot_probe(oracle_lib, L):
    """Q = 0 and a one-hot, large table cell (a, c): every query whose window contains the key
    at offset (a-L+1, c-L+1) attends (almost) only to it (pins sign, orientation and the
    peripheral cells, which get a single (query,key) pair per map)."""
    H, W, d = 11, 12, 4
    T = 2 * L - 1
    g = np.random.default_rng(L)
    v = g.standard_normal((1, 1, H, W, d))
    q = np.zeros_like(v)
    k = g.standard_normal(v.shape)
    for a, c in [(0, 0), (T - 1, T - 1), (0, T - 1), (L - 1, L - 1), (1, L + 1)]:
        rpb = np.zeros((1, T, T))
        rpb[0, a, c] = 400.0
        out, _ = oracle.na2d_forward(q, k, v, rpb, L, 0.5)
        hits = 0
        for i in range(H):
            for j in range(W):
                p, qq = i + a - (L - 1), j + c - (L - 1)
                si, sj = ref.window_start_argmin(i, H, L), ref.window_start_argmin(j, W, L)
                if si <= p < si + L and sj <= qq < sj + L:
                    hits += 1
                    np.testing.assert_allclose(out[0, 0, i, j], v[0, 0, p, qq], atol=1e-12)
                else:  # bias cell unused: plain window mean (Q = 0)
                    np.testing.assert_allclose(out[0, 0, i, j], v[0, 0, si:si + L, sj:sj + L].mean((0, 1)), atol=1e-12)
        assert hits >= 1


def test_reflection_symmetry(oracle_lib):
    """Flip Q,K,V along W and the table along its column axis => O flips (derived from
    start(n-1-i) = (n-L) - start(i))."""
    q, k, v, _, rpb = rand_problem(1, 2, 9, 11, 4, 5, seed=7)
    o, _ = oracle.na2d_forward(q, k, v, rpb, 5)
    f = lambda x: x[:, :, :, ::-1].copy()
    o2, _ = oracle.na2d_forward(f(q), f(k), f(v), rpb[:, :, ::-1].copy(), 5)
    np.testing.assert_allclose(o2, f(o), atol=1e-12)
    g = lambda x: x[:, :, ::-1].copy()
    o3, _ = oracle.na2d_forward(g(q), g(k), g(v), rpb[:, ::-1, :].copy(), 5)
    np.testing.assert_allclose(o3, g(o), atol=1e-12)


def test_translation_equivariance_and_locality(oracle_lib):
    L, ns = 5, 2
    q, k, v, _, rpb = rand_problem(1, 1, 12, 12, 4, L, seed=8)
    o, _ = oracle.na2d_forward(q, k, v, rpb, L)
    sh = lambda x: np.roll(x, (2, 3), axis=(2, 3))
    o2, _ = oracle.na2d_forward(sh(q), sh(k), sh(v), rpb, L)
    # interior queries of both frames (>= NS from every border, window not wrapping)
    for i in range(ns, 12 - ns - 2):
        for j in range(ns, 12 - ns - 3):
            np.testing.assert_allclose(o2[0, 0, i + 2, j + 3], o[0, 0, i, j], atol=1e-12)
    # locality: perturbing key/value pixel (a,b) only changes queries whose window holds it
    a, b = 5, 0
    k2, v2 = k.copy(), v.copy()
    k2[0, 0, a, b] += 1.0
    v2[0, 0, a, b] -= 2.0
    o3, _ = oracle.na2d_forward(q, k2, v2, rpb, L)
    for i in range(12):
        for j in range(12):
            si, sj = ref.window_start_argmin(i, 12, L), ref.window_start_argmin(j, 12, L)
            inside = si <= a < si + L and sj <= b < sj + L
            changed = np.abs(o3[0, 0, i, j] - o[0, 0, i, j]).max() > 0
            assert inside == changed


def test_errors(oracle_lib):
    q = np.zeros((1, 1, 4, 4, 2))
    for bad_L in (2, 4, 1, 0):
        with pytest.raises(oracle.OracleError):
            oracle.na2d_forward(q, q, q, None, bad_L)
    q[0, 0, 0, 0, 0] = np.inf
    with pytest.raises(oracle.OracleError):
        oracle.na2d_forward(q, np.ones_like(q), q, None, 3)


# ---------------------------------------------------------------- backward (a6-a10)

@pytest.mark.parametrize("H,W,L,with_bias", [(4, 5, 3, True), (6, 7, 5, True), (5, 5, 7, True), (7, 6, 3, False)])
def test_backward_matches_autograd_of_dense_formulation(oracle_lib, H, W, L, with_bias):
    import torch
    q, k, v, do, rpb = rand_problem(2, 2, H, W, 6, L, seed=H * W + L, with_bias=with_bias)
    g = oracle.na2d_backward(q, k, v, rpb, do, L, 6 ** -0.5)
    tq, tk, tv = (torch.from_numpy(x).requires_grad_() for x in (q, k, v))
    tb = torch.from_numpy(rpb).requires_grad_() if with_bias else None
    out, lse = ref.na2d_dense(tq, tk, tv, tb, L, 6 ** -0.5)
    out.backward(torch.from_numpy(do))
    np.testing.assert_allclose(g["out"], out.detach().numpy(), atol=1e-12)
    np.testing.assert_allclose(g["lse"], lse.detach().numpy(), atol=1e-12)
    np.testing.assert_allclose(g["dq"], tq.grad.numpy(), atol=1e-11)
    np.testing.assert_allclose(g["dk"], tk.grad.numpy(), atol=1e-11)
    np.testing.assert_allclose(g["dv"], tv.grad.numpy(), atol=1e-11)
    if with_bias:
        np.testing.assert_allclose(g["drpb"], tb.grad.numpy(), atol=1e-11)
    else:
        assert g["drpb"] is None


def test_backward_finite_differences(oracle_lib):
    """S:247 / S:569: central differences, h = 1e-5, relative error <= 1e-4."""
    L, hstep = 3, 1e-5
    for seed in range(3):
        q, k, v, do, rpb = rand_problem(1, 1, 4, 5, 6, L, seed=100 + seed)
        g = oracle.na2d_backward(q, k, v, rpb, do, L, 6 ** -0.5)
        loss = lambda qq, kk, vv, bb: float((oracle.na2d_forward(qq, kk, vv, bb, L, 6 ** -0.5)[0] * do).sum())
        rng = np.random.default_rng(seed)
        for name, arr in (("dq", q), ("dk", k), ("dv", v), ("drpb", rpb)):
            for _ in range(6):
                idx = tuple(rng.integers(0, s) for s in arr.shape)
                args = {"dq": [q, k, v, rpb], "dk": [q, k, v, rpb], "dv": [q, k, v, rpb], "drpb": [q, k, v, rpb]}[name]
                pos = {"dq": 0, "dk": 1, "dv": 2, "drpb": 3}[name]
                plus = [a.copy() for a in args]
                minus = [a.copy() for a in args]
                plus[pos][idx] += hstep
                minus[pos][idx] -= hstep
                fd = (loss(*plus) - loss(*minus)) / (2 * hstep)
                an = g[name][idx]
                assert abs(fd - an) <= 1e-4 * max(1.0, abs(an)), (name, idx, fd, an)


def test_gradient_identities(oracle_lib):
    """Per (b,h): sum over cells of dB = 0 (sum_m dS_m = 0 per query), sum_p dK_p = 0,
    sum_p dV_p = sum_ij dO_ij; dO = 0 => all gradients 0."""
    q, k, v, do, rpb = rand_problem(3, 2, 9, 8, 5, 5, seed=11)
    g = oracle.na2d_backward(q, k, v, rpb, do, 5)
    np.testing.assert_allclose(g["drpb"].sum(axis=(1, 2)), 0.0, atol=1e-11)
    np.testing.assert_allclose(g["dk"].sum(axis=(2, 3)), 0.0, atol=1e-11)
    np.testing.assert_allclose(g["dv"].sum(axis=(2, 3)), do.sum(axis=(2, 3)), atol=1e-11)
    z = oracle.na2d_backward(q, k, v, rpb, np.zeros_like(do), 5)
    for n in ("dq", "dk", "dv", "drpb"):
        assert np.all(z[n] == 0.0)


def test_gradients_equal_dense_sa_when_window_covers_map(oracle_lib):
    import torch
    q, k, v, do, _ = rand_problem(1, 1, 5, 5, 4, 7, seed=12, with_bias=False)
    g = oracle.na2d_backward(q, k, v, None, do, 7, 0.5)
    tq, tk, tv = (torch.from_numpy(x.reshape(25, 4)).requires_grad_() for x in (q, k, v))
    p = torch.softmax(tq @ tk.T * 0.5, -1)
    (p @ tv).backward(torch.from_numpy(do.reshape(25, 4)))
    for n, t in (("dq", tq), ("dk", tk), ("dv", tv)):
        np.testing.assert_allclose(g[n].reshape(25, 4), t.grad.numpy(), atol=1e-12)


def test_thread_count_determinism(oracle_lib):
    q, k, v, do, rpb = rand_problem(4, 3, 10, 9, 4, 5, seed=13)
    a = oracle.na2d_backward(q, k, v, rpb, do, 5, nthreads=1)
    b = oracle.na2d_backward(q, k, v, rpb, do, 5, nthreads=5)
    for n in a:
        assert np.array_equal(a[n], b[n]), n


# ---------------------------------------------------------------- row bands

def band_rows(H, G, L):
    """Owner rows and the K/V rows a band needs (global-coordinate clamp)."""
    out = []
    for r in range(G):
        r0, r1 = r * H // G, (r + 1) * H // G
        k0 = oracle.window_start(r0, H, L)
        k1 = oracle.window_start(r1 - 1, H, L) + oracle.window_len(H, L)
        out.append((r0, r1, k0, k1))
    return out


@pytest.mark.parametrize("H,G,L", [(20, 2, 7), (21, 3, 5), (16, 4, 3), (30, 4, 7)])
def test_band_split_equals_whole_map(oracle_lib, H, G, L):
    q, k, v, do, rpb = rand_problem(2, 2, H, 6, 4, L, seed=H + G)
    whole = oracle.na2d_backward(q, k, v, rpb, do, L)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    drpb = np.zeros_like(rpb)
    ns = (L - 1) // 2
    for r0, r1, k0, k1 in band_rows(H, G, L):
        assert k0 >= r0 - ns and k1 <= r1 + ns     # halo never exceeds NS rows (band >= L)
        out, lse = oracle.na2d_forward(q[:, :, r0:r1], k[:, :, k0:k1], v[:, :, k0:k1], rpb, L,
                                       H=H, q_row0=r0, kv_row0=k0)
        np.testing.assert_allclose(out, whole["out"][:, :, r0:r1], atol=1e-13)
        np.testing.assert_allclose(lse, whole["lse"][:, :, r0:r1], atol=1e-13)
        g = oracle.na2d_backward(q[:, :, r0:r1], k[:, :, k0:k1], v[:, :, k0:k1], rpb, do[:, :, r0:r1], L,
                                 H=H, q_row0=r0, kv_row0=k0)
        np.testing.assert_allclose(g["dq"], whole["dq"][:, :, r0:r1], atol=1e-12)
        dk[:, :, k0:k1] += g["dk"]
        dv[:, :, k0:k1] += g["dv"]
        drpb += g["drpb"]
    np.testing.assert_allclose(dk, whole["dk"], atol=1e-12)
    np.testing.assert_allclose(dv, whole["dv"], atol=1e-12)
    np.testing.assert_allclose(drpb, whole["drpb"], atol=1e-11)


def test_band_missing_rows_is_an_error(oracle_lib):
    q = np.zeros((1, 1, 4, 5, 2))
    with pytest.raises(oracle.OracleError):
        oracle.na2d_forward(q, np.zeros((1, 1, 4, 5, 2)), np.zeros((1, 1, 4, 5, 2)), None, 3,
                            H=12, q_row0=4, kv_row0=4)


# ---------------------------------------------------------------- inputs module

def test_inputs_are_bf16_and_sliceable():
    from na2d_inputs import bf16_round, bf16_bits
    s = Shape("t", 4, 2, 5, 6, 8, 3)
    a = make_inputs(s, seed=5)
    for n in ("q", "k", "v", "dout"):
        assert np.array_equal(bf16_round(a[n]), a[n])
        assert a[n].shape == (4, 2, 5, 6, 8)
    part = make_inputs(s, seed=5, batch_offset=1, batch_count=2)
    assert np.array_equal(part["q"], a["q"][1:3]) and np.array_equal(part["rpb"], a["rpb"])
    # RNE: 1 + 2^-8 is a tie between 1 and 1 + 2^-7 -> even (1.0); 1 + 3*2^-8 -> 1 + 2^-6
    x = np.array([1 + 2 ** -8, 1 + 3 * 2 ** -8, -2.5], np.float32)
    np.testing.assert_array_equal(bf16_round(x), np.array([1.0, 1 + 2 ** -6, -2.5], np.float32))
    assert bf16_bits(np.array([1.0], np.float32))[0] == 0x3F80


@pytest.mark.parametrize("L", [3, 5, 7, 9])
def test_inverse_neighbourhood_closed_form(oracle_lib, L):
    """The kernels' closed-form inverse neighbourhood (first/last query whose clamped window holds
    a key) equals brute-force enumeration over the oracle's windows, incl. bands [lo, hi)."""
    ns = (L - 1) // 2
    for n in range(1, 45):
        for lo, hi in [(0, n), (min(2, n - 1), n), (0, max(1, n - 3))]:
            for p in range(n):
                qs = [i for i in range(lo, hi) if oracle.window_start(i, n, L) <= p < oracle.window_start(i, n, L) + oracle.window_len(n, L)]
                cl = lo if (L >= n or p < L) else max(lo, p - ns)
                ch = hi - 1 if (L >= n or p >= n - L) else min(hi - 1, p + ns)
                if qs:
                    assert (cl, ch) == (qs[0], qs[-1]), (n, L, p, lo, hi)
                else:
                    assert cl > ch or not any(lo <= i < hi for i in range(cl, ch + 1)), (n, L, p, lo, hi)
