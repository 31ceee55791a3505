"""Host-side tests of the C ABI (-m "not gpu"): the library loads without a GPU, exports every
symbol include/na2d.h declares, and validates arguments synchronously (no launch happens on
an invalid call, so these run on a CPU-only machine)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def na2d():
    from paper_2204_07143_b200 import build
    build.build()
    import paper_2204_07143_b200 as m
    m.load_library()
    return m


def declared_functions():
    src = open(os.path.join(ROOT, "include", "na2d.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(na2d_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(na2d):
    names = declared_functions()
    assert len(names) >= 9, names
    lib = ctypes.CDLL(na2d.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(na2d.EXPORTS)
    assert lib.na2d_version() == 100


def test_problem_struct_matches_header(na2d):
    src = open(os.path.join(ROOT, "include", "na2d.h")).read()
    body = src[src.index("typedef struct {"):src.index("} na2d_problem;")]
    fields = re.findall(r"\b(?:int32_t|float)\s+(\w+);", body)
    assert fields == [f for f, _ in na2d.na2d_problem._fields_]


def P(na2d, **kw):
    base = dict(batch=1, heads=1, height=8, width=8, dim=32, kernel_size=3)
    base.update(kw)
    return na2d.make_problem(**base)


FAKE = 0x10000  # 16-byte aligned, never dereferenced: validation fails before any launch


@pytest.mark.parametrize("kw,status", [
    (dict(kernel_size=4), 2), (dict(kernel_size=1), 2), (dict(kernel_size=2), 2),
    (dict(height=0), 3), (dict(width=-1), 3), (dict(batch=0), 3), (dict(dim=0), 3),
    (dict(dtype=7), 4), (dict(dim=130), 5), (dict(dim=31), 5), (dict(kernel_size=33), 5),
    (dict(scale=0.0), 8), (dict(scale=float("inf")), 8), (dict(scale=float("nan")), 8), (dict(scale=-1.0), 8),
    # band: query rows [2, 6) of a 16-row map need K/V rows [0, 7) for L=3 -> [1, 7) held is not enough
    (dict(height=4, map_height=16, q_row0=2, kv_row0=2, kv_rows=5), 3),
    (dict(height=4, map_height=6, q_row0=4), 3),
])
def test_forward_validation(na2d, kw, status):
    p = P(na2d, **kw)
    lib = na2d.load_library()
    assert lib.na2d_forward(ctypes.byref(p), FAKE, FAKE, FAKE, None, FAKE, None, None) == status
    assert na2d.na2d_launch_count(p, 0) == -1
    assert na2d.na2d_kernel_family(p, 0) is None


def test_null_and_alignment(na2d):
    lib = na2d.load_library()
    p = P(na2d)
    assert lib.na2d_forward(None, FAKE, FAKE, FAKE, None, FAKE, None, None) == 1
    assert lib.na2d_forward(ctypes.byref(p), None, FAKE, FAKE, None, FAKE, None, None) == 1
    assert lib.na2d_forward(ctypes.byref(p), FAKE, FAKE, FAKE, None, None, None, None) == 1
    assert lib.na2d_forward(ctypes.byref(p), FAKE + 8, FAKE, FAKE, None, FAKE, None, None) == 6
    with pytest.raises(na2d.NA2DError) as e:
        na2d.na2d_forward(p, FAKE, FAKE + 2, FAKE, None, FAKE, None, None)
    assert e.value.status == 6


def test_backward_validation(na2d):
    lib = na2d.load_library()
    p = P(na2d)
    need = na2d.na2d_backward_workspace_bytes(p)
    assert need >= 64 * 4  # at least D (fp32 per query)
    args = [FAKE] * 7 + [FAKE, FAKE, FAKE]  # q k v rpb out lse dout dq dk dv
    # rpb given but drpb NULL
    assert lib.na2d_backward(ctypes.byref(p), *args, None, FAKE, need, None) == 8
    # workspace too small
    assert lib.na2d_backward(ctypes.byref(p), *args, FAKE, FAKE, need - 1, None) == 7
    # workspace NULL
    assert lib.na2d_backward(ctypes.byref(p), *args, FAKE, None, need, None) == 1
    # lse NULL
    a2 = list(args)
    a2[5] = None
    assert lib.na2d_backward(ctypes.byref(p), *a2, FAKE, FAKE, need, None) == 1
    assert na2d.na2d_backward_workspace_bytes(P(na2d, kernel_size=4)) == 0


def test_step_host_validation(na2d):
    p = P(na2d)
    assert na2d.na2d_step_host_workspace_bytes(p) > 0
    band = P(na2d, height=4, map_height=16, q_row0=4, kv_row0=2, kv_rows=8)
    assert na2d.na2d_step_host_workspace_bytes(band) == 0
    lib = na2d.load_library()
    assert lib.na2d_step_host(ctypes.byref(band), *([FAKE] * 12), FAKE, 1 << 30, None) == 3


def test_dispatch_families(na2d):
    # fp32 always takes the SIMT FFMA path (1e-4 relative parity forbids TF32)
    assert na2d.na2d_kernel_family(P(na2d, dtype=na2d.NA2D_F32, kernel_size=7, height=56, width=56), 0) == "simt"
    assert na2d.na2d_launch_count(P(na2d, dtype=na2d.NA2D_F32), 0) >= 1
    assert na2d.na2d_launch_count(P(na2d), 1) >= 1
    assert na2d.na2d_status_string(2).startswith("kernel_size")


def test_no_cpu_path(na2d):
    import torch
    q = torch.zeros(1, 1, 8, 8, 32, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="CUDA"):
        na2d.forward(q, q, q, None, 3)


def test_f16_accepted(na2d):
    """NA2D_F16 is a valid dtype on every path: validation passes and dispatch picks tcgen05 for
    the tensor-core shapes, SIMT otherwise (no device needed for these host-side queries)."""
    p = P(na2d, dtype=na2d.NA2D_F16, dim=64)
    assert na2d.na2d_launch_count(p, 0) >= 1
    assert na2d.na2d_kernel_family(p, 0) == "simt"
    assert na2d.na2d_status_string(4).startswith("dtype must be NA2D_BF16, NA2D_F32 or NA2D_F16")


@pytest.mark.parametrize("bad", ["k_width", "v_dtype", "rpb_bf16", "rpb_shape", "lse_shape", "dout_shape",
                                 "drpb_bf16", "drpb_missing"])
def test_torch_wrapper_validates_buffers(na2d, bad):
    """The C ABI cannot see buffer sizes: the torch wrappers reject any tensor whose shape or dtype
    does not match q's geometry (else an out-of-bounds device access), before the library is called."""
    import torch
    bf = torch.bfloat16
    q = torch.zeros(1, 2, 8, 8, 32, dtype=bf)
    k, v, dout = q.clone(), q.clone(), q.clone()
    rpb = torch.zeros(2, 5, 5)
    lse = torch.zeros(1, 2, 8, 8)
    grads = [q.clone(), q.clone(), q.clone(), rpb.clone()]
    if bad == "k_width":
        k = torch.zeros(1, 2, 8, 9, 32, dtype=bf)
    elif bad == "v_dtype":
        v = v.float()
    elif bad == "rpb_bf16":
        rpb = rpb.to(bf)
    elif bad == "rpb_shape":
        rpb = torch.zeros(2, 7, 7)
    elif bad == "lse_shape":
        lse = torch.zeros(1, 2, 8, 9)
    elif bad == "dout_shape":
        dout = torch.zeros(1, 2, 8, 8, 16, dtype=bf)
    elif bad == "drpb_bf16":
        grads[3] = grads[3].to(bf)
    elif bad == "drpb_missing":
        grads[3] = None
    with pytest.raises(ValueError, match="shape|dtype|drpb"):
        if bad in ("lse_shape", "dout_shape", "drpb_bf16", "drpb_missing"):
            na2d.backward(q, k, v, rpb, q, lse, dout, 3, grads=grads)
        else:
            na2d.forward(q, k, v, rpb, 3)
