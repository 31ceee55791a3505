"""The parity bound itself (tests/parity.py, R7 / R7b), on synthetic arrays (CPU)."""
import numpy as np
import pytest

from tests.parity import BF16_ATOL, compare, half_ulp


def _case(ref_val, err, dtype="bf16"):
    r = np.full((2, 1, 3, 3, 4), 0.5)
    r[0, 0, 1, 1, 2] = ref_val
    g = r.copy()
    g[0, 0, 1, 1, 2] += err
    return dict(out=g), dict(out=r), dtype


def test_half_ulp_values():
    assert half_ulp(np.array([1.0]), "bf16")[0] == 2.0 ** -8
    assert half_ulp(np.array([5.0]), "bf16")[0] == 2.0 ** -6
    assert half_ulp(np.array([5.0]), "f16")[0] == 2.0 ** -9


def test_strict_bound_below_four():
    compare(*_case(3.0, 0.0199))
    with pytest.raises(AssertionError):
        compare(*_case(3.0, 0.0201))
    with pytest.raises(AssertionError):  # the allowance never applies below |x| = 4
        compare(*_case(3.99, 0.03))


def test_output_rounding_allowance_from_four():
    compare(*_case(5.0, BF16_ATOL + 2.0 ** -6 - 1e-4))  # bf16 half-ULP in [4, 8) = 0.0156
    with pytest.raises(AssertionError):
        compare(*_case(5.0, BF16_ATOL + 2.0 ** -6 + 1e-4))
    with pytest.raises(AssertionError):  # fp16's half-ULP there is only 0.00195
        compare(*_case(5.0, 0.025, "f16"))


def test_other_elements_keep_the_strict_bound():
    got, ref, dt = _case(5.0, 0.03)
    got["out"][1, 0, 0, 0, 0] += 0.021  # an ordinary element just over 2e-2
    with pytest.raises(AssertionError):
        compare(got, ref, dt)


def test_fp32_outputs_get_no_allowance():
    r = {"out": np.zeros((1, 1, 8, 8, 1)), "lse": np.full((1, 1, 8, 8), 5.0)}
    g = {"out": r["out"], "lse": r["lse"] + 0.03}
    with pytest.raises(AssertionError, match="lse"):
        compare(g, r, "bf16")
