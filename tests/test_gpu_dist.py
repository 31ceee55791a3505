"""The multi-GPU partitions on the CUDA path (-m gpu): two ranks share the box's one GPU over gloo
(the driver's boxes have a single GPU), each runs its partition through the C ABI, and the
gathered results equal the fp64 oracle on the whole problem at the north-star tolerances:
row bands (K/V halo exchange, dK/dV halo partials returned and summed in fp32, dRPB all-reduce)
and batch x heads units with heads split across ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from na2d_inputs import Shape, make_inputs
from tests.parity import compare

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, mode, q_res):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2204_07143_b200 import dist as nd
    inp = make_inputs(shape, seed=41)
    L, scale = shape.kernel_size, shape.d ** -0.5
    cu = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().bfloat16()  # noqa: E731
    rpb = torch.from_numpy(inp["rpb"]).cuda()
    if mode == "band":
        band = nd.band_plan(shape.H, world, L)[rank]
        sl = slice(band.r0, band.r1)
        q, k, v, do = (cu(inp[n][:, :, sl]) for n in ("q", "k", "v", "dout"))
        out, lse, (k_ext, v_ext) = nd.band_forward(q, k, v, rpb, L, scale, band)
        dq, dk, dv, drpb = nd.band_backward(q, k_ext, v_ext, rpb, out, lse, do, L, scale, band)
        res = dict(out=out, lse=lse, dq=dq, dk=dk, dv=dv, drpb=drpb)
        q_res.put((rank, band.r0, band.r1, {n: x.float().cpu().numpy() for n, x in res.items()}))
    else:
        import paper_2204_07143_b200 as na2d
        q, k, v, do = (nd.unit_shard(torch.from_numpy(inp[n]), world, rank).cuda().bfloat16()
                       for n in ("q", "k", "v", "dout"))
        urpb = nd.unit_rpb(rpb, shape.B, world, rank)
        out, lse = na2d.forward(q, k, v, urpb, L, scale)
        dq, dk, dv, du = na2d.backward(q, k, v, urpb, out, lse, do, L, scale)
        drpb = nd.unit_drpb_to_heads(du, shape.heads, shape.B, world, rank)
        units = lambda x: x.reshape((-1,) + tuple(x.shape[2:]))  # noqa: E731  ([B', heads] or [1, units])
        res = dict(out=units(out), lse=units(lse), dq=units(dq), dk=units(dk), dv=units(dv), drpb=drpb)
        u0, u1 = nd.shard_range(shape.B * shape.heads, world, rank)
        q_res.put((rank, u0, u1, {n: x.float().cpu().numpy() for n, x in res.items()}))
    dist.barrier()
    dist.destroy_process_group()


def _run(shape, mode, world):
    ctx = mp.get_context("spawn")
    q_res = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, mode, q_res)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q_res.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_row_bands_cuda_match_whole_map(world):
    import oracle
    shape = Shape("bandgpu", 2, 2, 45, 37, 32, 7)
    inp = make_inputs(shape, seed=41)
    ref = oracle.na2d_backward(inp["q"], inp["k"], inp["v"], inp["rpb"], inp["dout"], 7, 32 ** -0.5)
    got = {n: np.zeros_like(ref[n]) for n in ("out", "lse", "dq", "dk", "dv")}
    for rank, r0, r1, part in _run(shape, "band", world):
        for n in ("out", "lse", "dq", "dk", "dv"):
            got[n][:, :, r0:r1] = part[n]
        got["drpb"] = part["drpb"]
    compare(got, ref, "bf16")


def test_units_split_heads_cuda():
    import oracle
    shape = Shape("unitgpu", 3, 2, 21, 26, 32, 7)  # 6 units on 4 ranks: heads split across ranks
    inp = make_inputs(shape, seed=41)
    ref = oracle.na2d_backward(inp["q"], inp["k"], inp["v"], inp["rpb"], inp["dout"], 7, 32 ** -0.5)
    flat = {n: ref[n].reshape((6,) + ref[n].shape[2:]) for n in ("out", "lse", "dq", "dk", "dv")}
    got = {n: np.zeros_like(flat[n]) for n in flat}
    for rank, u0, u1, part in _run(shape, "units", 4):
        for n in ("out", "lse", "dq", "dk", "dv"):
            got[n][u0:u1] = part[n]
        got["drpb"] = part["drpb"]
    ref2 = dict(flat, drpb=ref["drpb"])
    compare(got, ref2, "bf16", terms=3 * 21 * 26)
