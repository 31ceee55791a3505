"""The parity harness itself (-m "not gpu"): tolerances follow the north star, and a single
perturbed output element (fault injection) makes the comparison fail."""
import numpy as np
import pytest

from tests.parity import compare, tolerance


def test_tolerances():
    r = np.array([0.5, -3.0])
    assert tolerance("out", r, "bf16") == 2e-2
    # dRPB: literal 2e-2 on short reductions (small maps, config 1), 1e-3 relative on long ones
    assert tolerance("drpb", np.array([50.0]), "bf16") == 2e-2
    assert tolerance("drpb", np.array([50.0]), "bf16", terms=64) == 2e-2
    assert tolerance("drpb", np.array([50.0]), "bf16", terms=401408) == pytest.approx(5e-2)
    assert tolerance("drpb", np.array([0.1]), "bf16", terms=401408) == pytest.approx(1e-3)
    assert tolerance("dq", np.array([7.0]), "f32") == pytest.approx(7e-4)
    assert tolerance("dq", np.array([0.5]), "f32") == pytest.approx(1e-4)


def test_fault_injection_is_caught():
    g = np.random.default_rng(0)
    ref = {"out": g.standard_normal((2, 3, 4)), "drpb": g.standard_normal((1, 5, 5))}
    got = {k: v + 1e-3 for k, v in ref.items()}
    compare(got, ref, "bf16")
    bad = {k: v.copy() for k, v in got.items()}
    bad["out"][1, 2, 3] += 0.03
    with pytest.raises(AssertionError, match="out"):
        compare(bad, ref, "bf16")
    nan = {k: v.copy() for k, v in got.items()}
    nan["drpb"][0, 0, 0] = np.nan
    with pytest.raises(AssertionError, match="non-finite"):
        compare(nan, ref, "bf16")
    with pytest.raises(AssertionError):
        compare({"out": ref["out"][:1]}, {"out": ref["out"]}, "bf16")


def test_drpb_bound_follows_problem_size():
    """compare() reads B*H*W from the 5-D reference output: a dRPB error of 2.5e-2 fails on a
    small map (literal 2e-2) and passes on a long reduction with ||dRPB|| = 50 (5e-2)."""
    g = np.random.default_rng(1)
    for (B, H, W), ok in [((1, 8, 8), False), ((128, 56, 56), True)]:
        ref = {"out": np.zeros((B, 1, H, W, 1)), "drpb": np.full((1, 3, 3), 50.0)}
        got = {"out": ref["out"], "drpb": ref["drpb"] + 2.5e-2}
        if ok:
            compare(got, ref, "bf16")
        else:
            with pytest.raises(AssertionError, match="drpb"):
                compare(got, ref, "bf16")
