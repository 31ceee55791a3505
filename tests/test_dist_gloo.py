"""Multi-process host logic of the NA2D partitioning (-m "not gpu"): world size 2 on CPU with the
gloo backend, the fp64 oracle as the compute function.  Covers the row-band halo exchange
(forward K/V halos, backward dK/dV halo-partial return, dRPB all-reduce) and batch sharding with
the dRPB all-reduce, against the whole-map oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_forward(q, k, v, rpb, L, scale, *, map_height, q_row0, kv_row0):
    import oracle
    out, lse = oracle.na2d_forward(q.numpy(), k.numpy(), v.numpy(), None if rpb is None else rpb.numpy(), L, scale,
                                   H=map_height, q_row0=q_row0, kv_row0=kv_row0, nthreads=2)
    return torch.from_numpy(out), torch.from_numpy(lse)


def _oracle_backward(q, k, v, rpb, out, lse, dout, L, scale, *, map_height, q_row0, kv_row0):
    import oracle
    g = oracle.na2d_backward(q.numpy(), k.numpy(), v.numpy(), None if rpb is None else rpb.numpy(), dout.numpy(), L,
                             scale, H=map_height, q_row0=q_row0, kv_row0=kv_row0, nthreads=2)
    return (torch.from_numpy(g["dq"]), torch.from_numpy(g["dk"]), torch.from_numpy(g["dv"]),
            None if g["drpb"] is None else torch.from_numpy(g["drpb"]))


def _inputs(B, heads, H, W, d, L, seed):
    g = np.random.default_rng(seed)
    t = [torch.from_numpy(g.standard_normal((B, heads, H, W, d))) for _ in range(4)]
    rpb = torch.from_numpy(g.standard_normal((heads, 2 * L - 1, 2 * L - 1)) * np.sqrt(d))
    return t, rpb


def _band_worker(rank, world, port, shape, L, q_res):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_07143_b200 import dist as nd
    B, heads, H, W, d = shape
    (q, k, v, do), rpb = _inputs(B, heads, H, W, d, L, seed=17)
    band = nd.band_plan(H, world, L)[rank]
    sl = slice(band.r0, band.r1)
    qs, ks, vs, dos = (x[:, :, sl].contiguous() for x in (q, k, v, do))
    scale = d ** -0.5
    out, lse, (k_ext, v_ext) = nd.band_forward(qs, ks, vs, rpb, L, scale, band, forward_fn=_oracle_forward)
    dq, dk, dv, drpb = nd.band_backward(qs, k_ext, v_ext, rpb, out, lse, dos, L, scale, band,
                                        backward_fn=_oracle_backward)
    q_res.put((rank, band.r0, band.r1, out.numpy(), lse.numpy(), dq.numpy(), dk.numpy(), dv.numpy(), drpb.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shape,L,world", [((2, 2, 23, 9, 4), 7, 2), ((1, 2, 17, 12, 4), 5, 2), ((2, 1, 24, 7, 3), 3, 3)])
def test_row_band_split_matches_whole_map(shape, L, world):
    import oracle
    ctx = mp.get_context("spawn")
    q_res = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, shape, L, q_res)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q_res.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    B, heads, H, W, d = shape
    (q, k, v, do), rpb = _inputs(B, heads, H, W, d, L, seed=17)
    whole = oracle.na2d_backward(q.numpy(), k.numpy(), v.numpy(), rpb.numpy(), do.numpy(), L, d ** -0.5)
    for rank, r0, r1, out, lse, dq, dk, dv, drpb in res:
        np.testing.assert_allclose(out, whole["out"][:, :, r0:r1], atol=1e-12)
        np.testing.assert_allclose(lse, whole["lse"][:, :, r0:r1], atol=1e-12)
        np.testing.assert_allclose(dq, whole["dq"][:, :, r0:r1], atol=1e-11)
        np.testing.assert_allclose(dk, whole["dk"][:, :, r0:r1], atol=1e-11)
        np.testing.assert_allclose(dv, whole["dv"][:, :, r0:r1], atol=1e-11)
        np.testing.assert_allclose(drpb, whole["drpb"], atol=1e-10)


def _shard_worker(rank, world, port, q_res):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_07143_b200 import dist as nd
    B, heads, H, W, d, L = 5, 2, 9, 8, 4, 5
    (q, k, v, do), rpb = _inputs(B, heads, H, W, d, L, seed=23)
    b0, b1 = nd.shard_range(B, world, rank)
    sl = slice(b0, b1)
    dq, dk, dv, drpb = _oracle_backward(q[sl], k[sl], v[sl], rpb, None, None, do[sl], L, d ** -0.5, map_height=H,
                                        q_row0=0, kv_row0=0)
    nd.allreduce_drpb(drpb)
    q_res.put((rank, b0, b1, dq.numpy(), drpb.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_batch_shards_with_drpb_allreduce():
    import oracle
    ctx = mp.get_context("spawn")
    q_res = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q_res)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q_res.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (q, k, v, do), rpb = _inputs(5, 2, 9, 8, 4, 5, seed=23)
    whole = oracle.na2d_backward(q.numpy(), k.numpy(), v.numpy(), rpb.numpy(), do.numpy(), 5, 0.5)
    for rank, b0, b1, dq, drpb in res:
        np.testing.assert_allclose(dq, whole["dq"][b0:b1], atol=1e-12)
        np.testing.assert_allclose(drpb, whole["drpb"], atol=1e-10)


def test_band_plan_and_shards():
    from paper_2204_07143_b200 import dist as nd
    for H, world, L in [(200, 2, 7), (200, 4, 7), (200, 8, 7), (56, 4, 7), (23, 3, 7)]:
        bands = nd.band_plan(H, world, L)
        assert bands[0].r0 == 0 and bands[-1].r1 == H
        for a, b in zip(bands, bands[1:]):
            assert a.r1 == b.r0
        for bd in bands:
            assert 0 <= bd.top <= (L - 1) // 2 and 0 <= bd.bottom <= (L - 1) // 2
    with pytest.raises(ValueError):
        nd.band_plan(20, 4, 7)
    assert [nd.shard_range(10, 3, r) for r in range(3)] == [(0, 3), (3, 6), (6, 10)]


def _unit_worker(rank, world, port, shape, q_res):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_07143_b200 import dist as nd
    B, heads, H, W, d, L = shape
    (q, k, v, do), rpb = _inputs(B, heads, H, W, d, L, seed=29)
    qs, ks, vs, dos = (nd.unit_shard(x, world, rank) for x in (q, k, v, do))
    urpb = nd.unit_rpb(rpb, B, world, rank)
    dq, dk, dv, du = _oracle_backward(qs, ks, vs, urpb, None, None, dos, L, d ** -0.5, map_height=H, q_row0=0,
                                      kv_row0=0)
    drpb = nd.unit_drpb_to_heads(du, heads, B, world, rank)
    u0, u1 = nd.shard_range(B * heads, world, rank)
    units = lambda x: x.numpy().reshape((-1,) + tuple(x.shape[2:]))  # noqa: E731  ([B', heads] or [1, units])
    q_res.put((rank, u0, u1, units(dq), units(dk), drpb.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shape,world", [((3, 2, 9, 8, 4, 5), 2), ((1, 2, 10, 9, 4, 3), 2), ((2, 2, 9, 7, 4, 5), 3),
                                         ((4, 2, 9, 8, 4, 5), 2)])
def test_unit_shards_split_heads(shape, world):
    """batch x heads sharding by (b, h) units: a rank's units run as one batch of
    'heads' with per-unit RPB tables, or keep the [B', heads] layout when the range is whole batches;
    per-unit dRPB folds back onto the heads and all-reduces.  The cases include B < world (heads
    split across ranks), unit ranges starting mid-batch, and whole-batch ranges."""
    import oracle
    ctx = mp.get_context("spawn")
    q_res = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_unit_worker, args=(r, world, port, shape, q_res)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q_res.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    B, heads, H, W, d, L = shape
    (q, k, v, do), rpb = _inputs(B, heads, H, W, d, L, seed=29)
    whole = oracle.na2d_backward(q.numpy(), k.numpy(), v.numpy(), rpb.numpy(), do.numpy(), L, d ** -0.5)
    flat = lambda x: x.reshape((B * heads,) + x.shape[2:])  # noqa: E731
    for rank, u0, u1, dq, dk, drpb in res:
        np.testing.assert_allclose(dq, flat(whole["dq"])[u0:u1], atol=1e-12)
        np.testing.assert_allclose(dk, flat(whole["dk"])[u0:u1], atol=1e-12)
        np.testing.assert_allclose(drpb, whole["drpb"], atol=1e-10)
