"""The parity harness itself (-m "not gpu"): tolerances follow the north star, and a single
perturbed output element (fault injection) makes the comparison fail."""
import numpy as np
import pytest

from tests.parity import compare, tolerance


def test_tolerances():
    r = np.array([0.5, -3.0])
    assert tolerance("out", r, "bf16") == 2e-2
    assert tolerance("drpb", np.array([50.0]), "bf16") == pytest.approx(1.0)
    assert tolerance("drpb", np.array([0.1]), "bf16") == 2e-2
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
