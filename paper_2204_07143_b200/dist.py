"""Multi-GPU partitioning of NA2D: one process per GPU, torch.distributed (NCCL on
GPUs, gloo in the CPU tests) for the plumbing.  The kernels stay in libna2d; this module only plans
the partition and moves the few bytes that cross it.

* Batch x heads sharding -- every (b, h) map is independent.  Ranks hold contiguous
  batch shards; forward needs no communication; backward's only exchange is the all-reduce of the
  dRPB partial (all ranks share the heads' bias tables): heads * (2L-1)^2 * 4 bytes.
* Row bands -- for maps too large for one rank (COCO-shaped 200 x 336): rank r owns query rows
  [r0, r1) of every map.  Its queries' windows need K/V rows [wstart(r0), wstart(r1-1) + L), i.e.
  at most (L-1)/2 rows of each neighbour (band height >= L).  Forward: receive those halo rows
  (send/recv with ranks r-1 and r+1), run the band kernel in global coordinates.  Backward: run
  the band kernel over the extended K/V rows (dK/dV partials for the halo rows come from this
  rank's queries), send the halo partials back to their owners, add the received ones, and
  all-reduce dRPB.

Compute functions are injectable (``forward_fn``, ``backward_fn``) so the host logic is tested on
CPU with gloo and the fp64 oracle; the defaults call the CUDA library.
"""
from __future__ import annotations

import dataclasses

import torch
import torch.distributed as dist


def _wstart(i: int, n: int, L: int) -> int:
    if L >= n:
        return 0
    return min(max(i - (L - 1) // 2, 0), n - L)


# ------------------------------------------------------------------ batch x heads sharding

def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) of n units owned by `rank` (sizes differ by at most 1)."""
    return n * rank // world, n * (rank + 1) // world


def whole_batches(B: int, heads: int, world: int, rank: int) -> bool:
    """True if this rank's contiguous range of the B*heads (b, h) units is a range of whole batches."""
    u0, u1 = shard_range(B * heads, world, rank)
    return u0 % heads == 0 and u1 % heads == 0


def unit_shard(x: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """x: [B, heads, ...] -> this rank's contiguous range of the B*heads (b, h) units.  Units are
    independent maps.  A range of whole batches keeps the [B', heads, ...] layout (one bias
    table per head, shared by the batches); otherwise (heads split, e.g. B=2, 2 heads on 4 ranks) the
    range is returned as [1, units, ...], one "head" per unit with its own table (unit_rpb)."""
    B, heads = x.shape[:2]
    u0, u1 = shard_range(B * heads, world, rank)
    if whole_batches(B, heads, world, rank):
        return x[u0 // heads:u1 // heads].contiguous()
    return x.reshape(B * heads, *x.shape[2:])[u0:u1].unsqueeze(0).contiguous()


def unit_heads(B: int, heads: int, world: int, rank: int) -> torch.Tensor:
    """Head index of each unit of this rank's shard (for the per-unit RPB tables and dRPB)."""
    u0, u1 = shard_range(B * heads, world, rank)
    return torch.arange(u0, u1) % heads


def unit_rpb(rpb: torch.Tensor | None, B: int, world: int, rank: int) -> torch.Tensor | None:
    """The RPB tables the shard's kernels take: the heads' own [heads, 2L-1, 2L-1] for a range of
    whole batches, else one per unit [units, 2L-1, 2L-1] (a gather of the heads' tables)."""
    if rpb is None:
        return None
    if whole_batches(B, rpb.shape[0], world, rank):
        return rpb
    idx = unit_heads(B, rpb.shape[0], world, rank).to(rpb.device)
    return rpb.index_select(0, idx).contiguous()


def unit_drpb_to_heads(drpb_units: torch.Tensor | None, heads: int, B: int, world: int, rank: int,
                       out: torch.Tensor | None = None, group=None) -> torch.Tensor | None:
    """The shard's dRPB -> per-head sums (per-unit partials folded over this rank's units in ascending
    order; already per head for a range of whole batches), then the all-reduce over ranks."""
    if drpb_units is None:
        return None
    if whole_batches(B, heads, world, rank):
        acc = drpb_units if out is None else out.copy_(drpb_units)
        return allreduce_drpb(acc, group)
    idx = unit_heads(B, heads, world, rank).to(drpb_units.device)
    acc = torch.zeros((heads,) + tuple(drpb_units.shape[1:]), device=drpb_units.device, dtype=drpb_units.dtype) \
        if out is None else out.zero_()
    acc.index_add_(0, idx, drpb_units)
    return allreduce_drpb(acc, group)


def allreduce_drpb(drpb: torch.Tensor | None, group=None) -> torch.Tensor | None:
    """Sum the dRPB partials of all ranks in place (the only exchange of the sharded backward)."""
    if drpb is not None and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(drpb, op=dist.ReduceOp.SUM, group=group)
    return drpb


# ------------------------------------------------------------------ row bands

@dataclasses.dataclass(frozen=True)
class Band:
    rank: int
    world: int
    H: int
    L: int
    r0: int   # owned query / key rows [r0, r1)
    r1: int
    k0: int   # K/V rows the owned queries need [k0, k1)
    k1: int

    @property
    def top(self) -> int:     # halo rows received from rank-1 (its last rows)
        return self.r0 - self.k0

    @property
    def bottom(self) -> int:  # halo rows received from rank+1 (its first rows)
        return self.k1 - self.r1


def band_plan(H: int, world: int, L: int) -> list[Band]:
    """Equal row bands; every band must hold >= L rows so halos only reach adjacent ranks and
    never exceed (L-1)/2 rows."""
    bands = []
    for r in range(world):
        r0, r1 = H * r // world, H * (r + 1) // world
        if r1 - r0 < L:
            raise ValueError(f"band {r} has {r1 - r0} rows < kernel size {L}")
        k0 = _wstart(r0, H, L)
        k1 = _wstart(r1 - 1, H, L) + min(L, H)
        assert r0 - k0 <= (L - 1) // 2 and k1 - r1 <= (L - 1) // 2
        bands.append(Band(r, world, H, L, r0, r1, k0, k1))
    return bands


def _p2p(ops_spec, group=None):
    """Run [(isend|irecv, tensor, peer)] as one batch; with gloo (CPU tests, ranks sharing one GPU)
    CUDA tensors are staged through host memory, since gloo's point-to-point ops are CPU-only."""
    if not ops_spec:
        return
    gloo = dist.get_backend(group) == "gloo"
    staged, ops = [], []
    for kind, t, peer in ops_spec:
        x = t
        if gloo and t.is_cuda:
            x = t.cpu() if kind == "send" else torch.empty(t.shape, dtype=t.dtype)
            staged.append((t, x, kind))
        ops.append(dist.P2POp(dist.isend if kind == "send" else dist.irecv, x, peer, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    for t, x, kind in staged:
        if kind == "recv":
            t.copy_(x)


def _exchange_rows(own: torch.Tensor, band: Band, group=None) -> torch.Tensor:
    """own: [..., r1-r0, W, d] rows of this rank -> [..., k1-k0, W, d] with neighbour halos."""
    ext = torch.empty(own.shape[:-3] + (band.k1 - band.k0,) + own.shape[-2:], device=own.device, dtype=own.dtype)
    ext[..., band.top:band.top + own.shape[-3], :, :] = own
    exchange_halo(ext, band, group)
    return ext


def exchange_halo(ext: torch.Tensor, band: Band, group=None, bufs: dict | None = None) -> None:
    """ext: [..., k1-k0, W, d] holding this rank's own rows at [top, top + r1 - r0): fill its halo rows
    from the neighbours (and send them theirs).  NCCL point-to-point on NCCL's stream; the caller's
    stream waits for it (no host sync on GPUs).  `bufs` caches the contiguous send / receive buffers
    (a band's halo rows are strided across the outer B x heads dimension)."""
    rows = band.r1 - band.r0
    bufs = {} if bufs is None else bufs

    def buf(name, like):
        b = bufs.get(name)
        if b is None or b.shape != like.shape or b.dtype != like.dtype or b.device != like.device:
            b = bufs[name] = torch.empty(like.shape, dtype=like.dtype, device=like.device)
        return b

    spec, recvs = [], []
    prev, nxt = band.rank - 1, band.rank + 1
    # what the neighbours need from us: rank-1's bottom halo = our first rows; rank+1's top = our last
    if prev >= 0:
        need_prev = _neighbour(band, prev).bottom
        if need_prev:
            src = ext[..., band.top:band.top + need_prev, :, :]
            spec.append(("send", buf("s_prev", src).copy_(src), prev))
        if band.top:
            dst = ext[..., :band.top, :, :]
            r = buf("r_prev", dst)
            spec.append(("recv", r, prev))
            recvs.append((dst, r))
    if nxt < band.world:
        need_next = _neighbour(band, nxt).top
        if need_next:
            src = ext[..., band.top + rows - need_next:band.top + rows, :, :]
            spec.append(("send", buf("s_next", src).copy_(src), nxt))
        if band.bottom:
            dst = ext[..., band.top + rows:, :, :]
            r = buf("r_next", dst)
            spec.append(("recv", r, nxt))
            recvs.append((dst, r))
    _p2p(spec, group)
    for dst, r in recvs:
        dst.copy_(r)


def _return_partials(ext: torch.Tensor, band: Band, group=None) -> torch.Tensor:
    """ext: [..., k1-k0, W, d] partial gradients for the extended rows; send the halo rows back to
    their owners, add what the neighbours computed for our rows; returns [..., r1-r0, W, d] (>= fp32)."""
    acc_t = ext.dtype if ext.dtype == torch.float64 else torch.float32  # halo partials summed in >= fp32
    own = ext[..., band.top:band.top + (band.r1 - band.r0), :, :].to(acc_t)
    spec, recvs = [], []
    prev, nxt = band.rank - 1, band.rank + 1
    if prev >= 0:
        if band.top:
            spec.append(("send", ext[..., :band.top, :, :].to(acc_t).contiguous(), prev))
        nb = _neighbour(band, prev).bottom  # rank-1 computed partials for our first nb rows
        if nb:
            buf = torch.empty_like(own[..., :nb, :, :])
            spec.append(("recv", buf, prev))
            recvs.append((0, buf))
    if nxt < band.world:
        if band.bottom:
            spec.append(("send", ext[..., ext.shape[-3] - band.bottom:, :, :].to(acc_t).contiguous(), nxt))
        nt = _neighbour(band, nxt).top  # rank+1 computed partials for our last nt rows
        if nt:
            buf = torch.empty_like(own[..., :nt, :, :])
            spec.append(("recv", buf, nxt))
            recvs.append((own.shape[-3] - nt, buf))
    _p2p(spec, group)
    for off, buf in recvs:
        own[..., off:off + buf.shape[-3], :, :] += buf
    return own


def _neighbour(band: Band, r: int) -> Band:
    return band_plan(band.H, band.world, band.L)[r]


def _cuda_forward(q, k, v, rpb, L, scale, *, map_height, q_row0, kv_row0):
    from . import forward
    return forward(q, k, v, rpb, L, scale, map_height=map_height, q_row0=q_row0, kv_row0=kv_row0)


def _cuda_backward(q, k, v, rpb, out, lse, dout, L, scale, *, map_height, q_row0, kv_row0):
    from . import backward
    return backward(q, k, v, rpb, out, lse, dout, L, scale, map_height=map_height, q_row0=q_row0,
                    kv_row0=kv_row0)


def band_forward(q, k, v, rpb, L: int, scale: float | None, band: Band, group=None, forward_fn=None):
    """q, k, v: this rank's own rows [B, heads, r1-r0, W, d].  Returns (out, lse) for own rows."""
    fn = forward_fn or _cuda_forward
    k_ext = _exchange_rows(k, band, group)
    v_ext = _exchange_rows(v, band, group)
    out, lse = fn(q, k_ext, v_ext, rpb, L, scale, map_height=band.H, q_row0=band.r0, kv_row0=band.k0)
    return out, lse, (k_ext, v_ext)


def band_backward(q, k_ext, v_ext, rpb, out, lse, dout, L: int, scale: float | None, band: Band, group=None,
                  backward_fn=None):
    """Backward of a band given the extended K/V from band_forward.  Returns (dq, dk, dv, drpb) for
    own rows, in q's dtype: the halo rows' dK / dV partials (this rank's queries) go back to their
    owners and are summed with the owners' own partials in fp32 before the one rounding to the
    output type; drpb all-reduced."""
    fn = backward_fn or _cuda_backward
    dq, dk_ext, dv_ext, drpb = fn(q, k_ext, v_ext, rpb, out, lse, dout, L, scale, map_height=band.H,
                                  q_row0=band.r0, kv_row0=band.k0)
    dk = _return_partials(dk_ext, band, group).to(q.dtype)
    dv = _return_partials(dv_ext, band, group).to(q.dtype)
    allreduce_drpb(drpb, group)
    return dq, dk, dv, drpb
