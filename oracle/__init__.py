"""fp64 CPU oracle for 2D Neighborhood Attention (arXiv 2204.07143, Eq. 2).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  It shares no code with
the CUDA path (``paper_2204_07143_b200``) and never imports it; the CUDA path never imports
this package.

Contents
--------
* ``na2d_oracle.c``  -- the oracle proper: plain fp64 C loops that follow Eq. 2,
  the clamped neighbourhood rho and the analytic backward.
  Loaded here through ctypes (compiled on first use with gcc, or by ``build()``).
* ``reference.py``   -- independent NumPy formulations used to pin the C oracle:
  masked dense self-attention (Eq. 1 + mask), Appendix A unfold + replicate padding,
  pure-Python loops for tiny maps.

Parity status: every function here is pinned by tests in ``tests/test_oracle.py``
(no "parity unpinned" functions except the two conventions listed in DESIGN.md R1/R4,
which are pinned by the RPB probe / reflection tests only).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "na2d_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libna2d_oracle.so")
_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile ``libna2d_oracle.so`` with gcc (plain -O2, no fast-math: fp64 IEEE)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            I, D, P = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
            lib.na2d_oracle_window_start.argtypes = [I, I, I]
            lib.na2d_oracle_window_start.restype = I
            lib.na2d_oracle_window_len.argtypes = [I, I]
            lib.na2d_oracle_window_len.restype = I
            lib.na2d_oracle_rel_index.argtypes = [I, I, I]
            lib.na2d_oracle_rel_index.restype = I
            lib.na2d_oracle_forward_band.argtypes = [I] * 6 + [D] + [I] * 4 + [P] * 6 + [I]
            lib.na2d_oracle_forward_band.restype = I
            lib.na2d_oracle_backward_band.argtypes = [I] * 6 + [D] + [I] * 4 + [P] * 11 + [I]
            lib.na2d_oracle_backward_band.restype = I
            _lib = lib
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class OracleError(RuntimeError):
    pass


_ERRS = {1: "bad argument (dims, or L not odd >= 3)", 2: "band does not supply a needed K/V row",
         3: "non-finite logits"}


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def window_start(i: int, n: int, L: int) -> int:
    """rho along one axis: start = clamp(i-(L-1)/2, 0, n-L); 0 if L>=n."""
    return _load().na2d_oracle_window_start(i, n, L)


def window_len(n: int, L: int) -> int:
    return _load().na2d_oracle_window_len(n, L)


def rel_index(i: int, p: int, L: int) -> int:
    """RPB index along one axis: key - query + L - 1."""
    return _load().na2d_oracle_rel_index(i, p, L)


def na2d_forward(q, k, v, rpb, kernel_size: int, inv_scale: float | None = None, *,
                 H: int | None = None, q_row0: int = 0, kv_row0: int = 0, nthreads: int | None = None):
    """Eq. 2 forward in fp64.  q: [B,heads,q_rows,W,d]; k,v: [B,heads,kv_rows,W,d];
    rpb: [heads,2L-1,2L-1] or None.  Returns (out [B,heads,q_rows,W,d], lse [B,heads,q_rows,W])."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    B, heads, q_rows, W, d = q.shape
    kv_rows = k.shape[2]
    H = q_rows if H is None else H
    if inv_scale is None:
        inv_scale = d ** -0.5
    rpb = None if rpb is None else _f64(rpb)
    out = np.empty_like(q)
    lse = np.empty(q.shape[:4], np.float64)
    rc = _load().na2d_oracle_forward_band(B, heads, H, W, d, kernel_size, float(inv_scale),
                                          q_row0, q_rows, kv_row0, kv_rows,
                                          _ptr(q), _ptr(k), _ptr(v), _ptr(rpb), _ptr(out), _ptr(lse),
                                          nthreads or default_threads())
    if rc:
        raise OracleError(_ERRS.get(rc, str(rc)))
    return out, lse


def na2d_backward(q, k, v, rpb, dout, kernel_size: int, inv_scale: float | None = None, *,
                  H: int | None = None, q_row0: int = 0, kv_row0: int = 0, nthreads: int | None = None):
    """Analytic backward of Eq. 2 in fp64.  Returns dict(out, lse, dq, dk, dv, drpb)."""
    q, k, v, dout = _f64(q), _f64(k), _f64(v), _f64(dout)
    B, heads, q_rows, W, d = q.shape
    kv_rows = k.shape[2]
    H = q_rows if H is None else H
    if inv_scale is None:
        inv_scale = d ** -0.5
    rpb = None if rpb is None else _f64(rpb)
    T = 2 * kernel_size - 1
    out = np.empty_like(q)
    lse = np.empty(q.shape[:4], np.float64)
    dq = np.empty_like(q)
    dk = np.empty_like(k)
    dv = np.empty_like(v)
    drpb = np.empty((heads, T, T), np.float64) if rpb is not None else None
    rc = _load().na2d_oracle_backward_band(B, heads, H, W, d, kernel_size, float(inv_scale),
                                           q_row0, q_rows, kv_row0, kv_rows,
                                           _ptr(q), _ptr(k), _ptr(v), _ptr(rpb), _ptr(dout),
                                           _ptr(out), _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv),
                                           _ptr(drpb), nthreads or default_threads())
    if rc:
        raise OracleError(_ERRS.get(rc, str(rc)))
    return dict(out=out, lse=lse, dq=dq, dk=dk, dv=dv, drpb=drpb)
