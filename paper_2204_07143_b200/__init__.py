"""B200-native 2D Neighborhood Attention (arXiv 2204.07143) -- thin Python binding.

Every step of the path runs in ``libna2d.so`` (hand-written sm_100a CUDA kernels behind the
C ABI in ``include/na2d.h``).  This module only marshals arguments: torch supplies device
memory and the current CUDA stream.  There is no CPU fallback: if the library is missing, or a
tensor is not on a CUDA device, calls raise.

Low level (same names as the C ABI, integer device pointers):
    na2d_forward, na2d_backward, na2d_backward_workspace_bytes, na2d_step_host,
    na2d_step_host_workspace_bytes, na2d_launch_count, na2d_kernel_family, na2d_status_string
Torch level:
    forward(q, k, v, rpb, kernel_size, scale=None) -> (out, lse)
    backward(q, k, v, rpb, out, lse, dout, kernel_size, scale=None) -> (dq, dk, dv, drpb)
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libna2d.so")

NA2D_BF16, NA2D_F32, NA2D_F16 = 0, 1, 2
_STATUS = ["ok", "null pointer", "kernel size", "shape", "dtype", "unsupported", "alignment", "workspace",
           "invalid argument", "cuda"]


class NA2DError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        msg = f"{what}: status {status} ({na2d_status_string(status)})"
        if status == 9:
            msg += ": " + load_library().na2d_last_cuda_error().decode()
        super().__init__(msg)


class na2d_problem(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("heads", ctypes.c_int32), ("height", ctypes.c_int32),
                ("width", ctypes.c_int32), ("dim", ctypes.c_int32), ("kernel_size", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("scale", ctypes.c_float), ("map_height", ctypes.c_int32),
                ("q_row0", ctypes.c_int32), ("kv_row0", ctypes.c_int32), ("kv_rows", ctypes.c_int32)]


EXPORTS = ("na2d_status_string", "na2d_version", "na2d_forward", "na2d_backward_workspace_bytes",
           "na2d_backward", "na2d_step_host_workspace_bytes", "na2d_step_host", "na2d_launch_count",
           "na2d_kernel_family", "na2d_profile_enable", "na2d_profile_read", "na2d_last_cuda_error",
           "na2d_debug_set_trace", "na2d_paper_attn_bytes", "na2d_paper_forward", "na2d_paper_backward")

_lib = None


def load_library():
    """Load libna2d.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with `python -m paper_2204_07143_b200.build` "
                          "(no CPU or eager fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    P, PP, VP, SZ = ctypes.POINTER(na2d_problem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t
    lib.na2d_status_string.argtypes = [ctypes.c_int]
    lib.na2d_status_string.restype = ctypes.c_char_p
    lib.na2d_version.restype = ctypes.c_int
    lib.na2d_forward.argtypes = [P] + [VP] * 7
    lib.na2d_forward.restype = ctypes.c_int
    lib.na2d_backward_workspace_bytes.argtypes = [P]
    lib.na2d_backward_workspace_bytes.restype = SZ
    lib.na2d_backward.argtypes = [P] + [VP] * 12 + [SZ, VP]
    lib.na2d_backward.restype = ctypes.c_int
    lib.na2d_step_host_workspace_bytes.argtypes = [P]
    lib.na2d_step_host_workspace_bytes.restype = SZ
    lib.na2d_step_host.argtypes = [P] + [VP] * 12 + [SZ, VP]
    lib.na2d_step_host.restype = ctypes.c_int
    lib.na2d_launch_count.argtypes = [P, ctypes.c_int]
    lib.na2d_launch_count.restype = ctypes.c_int
    lib.na2d_kernel_family.argtypes = [P, ctypes.c_int]
    lib.na2d_kernel_family.restype = ctypes.c_char_p
    lib.na2d_last_cuda_error.restype = ctypes.c_char_p
    lib.na2d_debug_set_trace.argtypes = [ctypes.c_void_p]
    lib.na2d_paper_attn_bytes.argtypes = [P]
    lib.na2d_paper_attn_bytes.restype = SZ
    lib.na2d_paper_forward.argtypes = [P] + [VP] * 8
    lib.na2d_paper_forward.restype = ctypes.c_int
    lib.na2d_paper_backward.argtypes = [P] + [VP] * 11
    lib.na2d_paper_backward.restype = ctypes.c_int
    lib.na2d_debug_set_trace.restype = ctypes.c_int
    lib.na2d_profile_enable.argtypes = [ctypes.c_int]
    lib.na2d_profile_enable.restype = ctypes.c_int
    lib.na2d_profile_read.argtypes = [ctypes.c_char_p, SZ, ctypes.POINTER(ctypes.c_float),
                                      ctypes.POINTER(ctypes.c_int), ctypes.c_int]
    lib.na2d_profile_read.restype = ctypes.c_int
    _lib = lib
    return lib


def make_problem(batch, heads, height, width, dim, kernel_size, dtype=NA2D_BF16, scale=None, *,
                 map_height=0, q_row0=0, kv_row0=0, kv_rows=0) -> na2d_problem:
    if scale is None:
        scale = dim ** -0.5 if dim > 0 else 1.0
    return na2d_problem(batch, heads, height, width, dim, kernel_size, dtype, float(scale), map_height, q_row0,
                        kv_row0, kv_rows)


# ------------------------------------------------------------------ C ABI, same names

def na2d_status_string(status: int) -> str:
    return load_library().na2d_status_string(status).decode()


def _check(status: int, what: str):
    if status != 0:
        raise NA2DError(status, what)


def na2d_forward(p: na2d_problem, q: int, k: int, v: int, rpb: int | None, out: int, lse: int | None,
                 stream: int | None) -> None:
    _check(load_library().na2d_forward(ctypes.byref(p), q, k, v, rpb, out, lse, stream), "na2d_forward")


def na2d_backward_workspace_bytes(p: na2d_problem) -> int:
    return load_library().na2d_backward_workspace_bytes(ctypes.byref(p))


def na2d_backward(p, q, k, v, rpb, out, lse, dout, dq, dk, dv, drpb, workspace, workspace_bytes, stream) -> None:
    _check(load_library().na2d_backward(ctypes.byref(p), q, k, v, rpb, out, lse, dout, dq, dk, dv, drpb,
                                        workspace, workspace_bytes, stream), "na2d_backward")


def na2d_step_host_workspace_bytes(p: na2d_problem) -> int:
    return load_library().na2d_step_host_workspace_bytes(ctypes.byref(p))


def na2d_step_host(p, q, k, v, rpb, dout, out, lse, dq, dk, dv, drpb, workspace, workspace_bytes, stream) -> None:
    _check(load_library().na2d_step_host(ctypes.byref(p), q, k, v, rpb, dout, out, lse, dq, dk, dv, drpb,
                                         workspace, workspace_bytes, stream), "na2d_step_host")


def na2d_launch_count(p: na2d_problem, which: int) -> int:
    return load_library().na2d_launch_count(ctypes.byref(p), which)


def na2d_kernel_family(p: na2d_problem, which: int) -> str | None:
    r = load_library().na2d_kernel_family(ctypes.byref(p), which)
    return None if r is None else r.decode()


def na2d_profile_enable(on: bool) -> None:
    _check(load_library().na2d_profile_enable(1 if on else 0), "na2d_profile_enable")


def na2d_profile_read() -> dict:
    """{kernel name: (total_ms, launches)} recorded since na2d_profile_enable(True)."""
    lib = load_library()
    n = 64
    names = ctypes.create_string_buffer(8192)
    ms = (ctypes.c_float * n)()
    cnt = (ctypes.c_int * n)()
    k = lib.na2d_profile_read(names, 8192, ms, cnt, n)
    if k < 0:
        raise NA2DError(9, "na2d_profile_read")
    out, parts = {}, names.raw.split(b"\0")
    for i in range(min(k, n)):
        out[parts[i].decode()] = (float(ms[i]), int(cnt[i]))
    return out


# ------------------------------------------------------------------ torch convenience layer

def _dtype_code(t):
    import torch
    if t.dtype == torch.bfloat16:
        return NA2D_BF16
    if t.dtype == torch.float32:
        return NA2D_F32
    if t.dtype == torch.float16:
        return NA2D_F16
    raise TypeError(f"unsupported dtype {t.dtype} (bf16, fp16 or fp32)")


def _dev(t, name):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _stream(t):
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


def _expect(t, name, shape, dtype, device):
    """The C ABI cannot see buffer sizes: every tensor's shape, dtype and device is checked here,
    before the library is called, so a mismatch raises instead of reading or writing out of bounds."""
    if t is None:
        return
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if t.device != device:
        raise ValueError(f"{name}: on {t.device}, expected {device} (the device of q)")


def _validate(q, k, v, rpb, kernel_size, **named):
    """q [B,heads,H,W,d]; k, v [B,heads,kv_rows,W,d] (kv_rows = H unless a row band); rpb fp32
    [heads,2L-1,2L-1]; named: dout/out like q, lse fp32 [B,heads,H,W], dq like q, dk/dv like k,
    drpb like rpb."""
    import torch
    if q.dim() != 5:
        raise ValueError(f"q: expected [B,heads,H,W,d], got shape {tuple(q.shape)}")
    B, heads, H, W, d = q.shape
    dev, dt = q.device, q.dtype
    kshape = (B, heads, k.shape[2] if k.dim() == 5 else -1, W, d)
    _expect(k, "k", kshape, dt, dev)
    _expect(v, "v", kshape, dt, dev)
    T = 2 * int(kernel_size) - 1
    _expect(rpb, "rpb", (heads, T, T), torch.float32, dev)
    like = {"dout": (q.shape, dt), "out": (q.shape, dt), "dq": (q.shape, dt), "lse": (q.shape[:4], torch.float32),
            "dk": (kshape, dt), "dv": (kshape, dt), "drpb": ((heads, T, T), torch.float32)}
    for n, t in named.items():
        shape, tdt = like[n]
        _expect(t, n, shape, tdt, dev)
    if (rpb is None) != (named.get("drpb", rpb) is None):
        raise ValueError("drpb must be given exactly when rpb is given")
    if not q.is_cuda:
        raise ValueError("q must be a CUDA tensor (no CPU path exists)")


def problem_for(q, k, kernel_size, scale=None, *, map_height=0, q_row0=0, kv_row0=0) -> na2d_problem:
    B, heads, H, W, d = q.shape
    return make_problem(B, heads, H, W, d, kernel_size, _dtype_code(q), scale, map_height=map_height,
                        q_row0=q_row0, kv_row0=kv_row0, kv_rows=k.shape[2])


def forward(q, k, v, rpb, kernel_size: int, scale: float | None = None, *, map_height=0, q_row0=0, kv_row0=0,
            out=None, lse=None):
    """Eq. 2 forward.  q: [B,heads,H,W,d] (bf16 or fp32, CUDA); k, v: [B,heads,kv_rows,W,d];
    rpb: [heads,2L-1,2L-1] fp32 or None.  Returns (out, lse fp32 [B,heads,H,W])."""
    import torch
    _validate(q, k, v, rpb, kernel_size, out=out, lse=lse)
    p = problem_for(q, k, kernel_size, scale, map_height=map_height, q_row0=q_row0, kv_row0=kv_row0)
    with torch.cuda.device(q.device):  # the library launches on the current device
        out = torch.empty_like(q) if out is None else out
        lse = torch.empty(q.shape[:4], device=q.device, dtype=torch.float32) if lse is None else lse
        na2d_forward(p, _dev(q, "q"), _dev(k, "k"), _dev(v, "v"), _dev(rpb, "rpb"), _dev(out, "out"),
                     _dev(lse, "lse"), _stream(q))
    return out, lse


def backward(q, k, v, rpb, out, lse, dout, kernel_size: int, scale: float | None = None, *, map_height=0,
             q_row0=0, kv_row0=0, workspace=None, grads=None):
    """Analytic backward of Eq. 2.  Returns (dq, dk, dv, drpb or None)."""
    import torch
    if grads is None:
        _validate(q, k, v, rpb, kernel_size, out=out, lse=lse, dout=dout)
    else:
        dq, dk, dv, drpb = grads
        _validate(q, k, v, rpb, kernel_size, out=out, lse=lse, dout=dout, dq=dq, dk=dk, dv=dv, drpb=drpb)
    if workspace is not None and (workspace.device != q.device or workspace.dtype != torch.uint8):
        raise ValueError("workspace must be a uint8 tensor on the device of q")
    p = problem_for(q, k, kernel_size, scale, map_height=map_height, q_row0=q_row0, kv_row0=kv_row0)
    with torch.cuda.device(q.device):  # the library launches on the current device
        nbytes = na2d_backward_workspace_bytes(p)
        if workspace is None or workspace.numel() < nbytes:
            workspace = torch.empty(max(nbytes, 16), device=q.device, dtype=torch.uint8)
        if grads is None:
            dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
            drpb = torch.empty_like(rpb) if rpb is not None else None
        na2d_backward(p, _dev(q, "q"), _dev(k, "k"), _dev(v, "v"), _dev(rpb, "rpb"), _dev(out, "out"),
                      _dev(lse, "lse"), _dev(dout, "dout"), _dev(dq, "dq"), _dev(dk, "dk"), _dev(dv, "dv"),
                      _dev(drpb, "drpb"), _dev(workspace, "workspace"), workspace.numel(), _stream(q))
    return dq, dk, dv, drpb


def paper_forward(q, k, v, rpb, kernel_size: int, scale: float | None = None):
    """The paper's unfused decomposition: QK+RPB -> softmax -> AV, materialising the
    attention weights.  Returns (out, lse, attn [B,heads,H,W,Lh*Lw] fp32)."""
    import torch
    _validate(q, k, v, rpb, kernel_size)
    if k.shape[2] != q.shape[2]:
        raise ValueError("the paper decomposition takes whole maps (k, v rows == q rows)")
    p = problem_for(q, k, kernel_size, scale)
    nwin = min(kernel_size, q.shape[2]) * min(kernel_size, q.shape[3])
    out = torch.empty_like(q)
    lse = torch.empty(q.shape[:4], device=q.device, dtype=torch.float32)
    attn = torch.empty(q.shape[:4] + (nwin,), device=q.device, dtype=torch.float32)
    with torch.cuda.device(q.device):
        _check(load_library().na2d_paper_forward(ctypes.byref(p), _dev(q, "q"), _dev(k, "k"), _dev(v, "v"),
                                                 _dev(rpb, "rpb"), _dev(out, "out"), _dev(lse, "lse"),
                                                 _dev(attn, "attn"), _stream(q)), "na2d_paper_forward")
    return out, lse, attn


def paper_backward(q, k, v, rpb, attn, dout, kernel_size: int, scale: float | None = None, dS=None):
    """Gradients of the unfused decomposition from its stored attention weights."""
    import torch
    _validate(q, k, v, rpb, kernel_size, dout=dout)
    if k.shape[2] != q.shape[2]:
        raise ValueError("the paper decomposition takes whole maps (k, v rows == q rows)")
    nwin = min(kernel_size, q.shape[2]) * min(kernel_size, q.shape[3])
    _expect(attn, "attn", q.shape[:4] + (nwin,), torch.float32, q.device)
    _expect(dS, "dS", q.shape[:4] + (nwin,), torch.float32, q.device)
    p = problem_for(q, k, kernel_size, scale)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    drpb = torch.empty_like(rpb) if rpb is not None else None
    dS = torch.empty_like(attn) if dS is None else dS
    with torch.cuda.device(q.device):
        _check(load_library().na2d_paper_backward(ctypes.byref(p), _dev(q, "q"), _dev(k, "k"), _dev(v, "v"),
                                                  _dev(dout, "dout"), _dev(attn, "attn"), _dev(dS, "dS"),
                                                  _dev(dq, "dq"), _dev(dk, "dk"), _dev(dv, "dv"),
                                                  _dev(drpb, "drpb"), _stream(q)), "na2d_paper_backward")
    return dq, dk, dv, drpb
