#!/usr/bin/env python
"""NA2D forward + backward benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl na2d|reference]

One step = the whole hot path: na2d_forward + na2d_backward over one
batch of the workload (default: NAT-Tiny stage 1, B=128, heads=2, 56x56, d=32, k=7, bf16), plus,
for N > 1, the NCCL all-reduce of the dRPB partials (every rank holds a different batch shard of
the same heads: weak scaling, per-rank batch fixed).  Inputs are resident in HBM before the
timed region; two input sets (205 MB each, > 126 MB L2) alternate between steps so no step
reads the previous step's inputs from L2.

Printed (rank 0, one JSON line): value = whole-job algorithmic TFLOP/s (4 N k^2 d fwd +
8 N k^2 d bwd flops, N = query-heads) over the max-over-ranks device time; roofline of the
dominant kernel (CUDA events around each launch, on the launching stream); cpu_baseline (the
fp64 oracle on a bounded sample, host cores); e2e through the host-buffer C-ABI entry point
(na2d_step_host: H2D + fwd + bwd + D2H); clocks sampled during the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from na2d_inputs import CONFIGS, EXTRA_WORKLOADS, Shape, make_inputs  # noqa: E402

METRIC = "NA2D fwd+bwd TFLOP/s and % of B200 roofline at 1/2/4/8 GPUs, NAT-Tiny k=7"
UNIT = "TFLOP/s"
DEFAULT_CONFIG = "cfg2_nat_tiny_s1"


def flops(shape: Shape, units: int | None = None) -> tuple[float, float]:
    """Algorithmic flops: fwd 4 N kh kw d, bwd 8 N kh kw d."""
    kh, kw = min(shape.kernel_size, shape.H), min(shape.kernel_size, shape.W)
    n = (shape.units if units is None else units) * shape.H * shape.W
    return 4.0 * n * kh * kw * shape.d, 8.0 * n * kh * kw * shape.d


def alg_bytes_per_query(kernel: str, d: int, s: int) -> float | None:
    """Algorithmic HBM bytes per query-head for each kernel."""
    if kernel.startswith("na2d_fwd"):
        return 4 * d * s + 4                  # read q,k,v; write out; write lse
    if kernel == "na2d_bwd_delta":
        return 2 * d * s + 4                  # read out,dout; write D
    if kernel.startswith("na2d_bwd_dq"):
        return 4 * d * s + 8 + d * s          # read q,k,v,dout,lse,D; write dq
    if kernel.startswith("na2d_bwd_dkdv"):
        return 4 * d * s + 8 + 2 * d * s      # read q,k,v,dout,lse,D; write dk,dv
    return None


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clocks / clock-event (throttle) reasons sampled while the timed region runs: NVML polled
    every ~0.5 ms by a helper process (a timed region of 20 steps lasts only ~8 ms), nvidia-smi
    every 200 ms if NVML is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x for x in vis.split(",") if x.strip()]
        self.index = int(ids[index]) if index < len(ids) and ids[index].strip().isdigit() else index
        self.rows: list[tuple] = []
        self._stop = threading.Event()
        self._t = None

    POLL = ("import sys, time, pynvml as nv\n"
            "nv.nvmlInit(); h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))\n"
            "mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)\n"
            "rs = getattr(nv, 'nvmlDeviceGetCurrentClocksEventReasons', None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons\n"
            "while True:\n"
            "    print(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx, rs(h), flush=True)\n"
            "    time.sleep(0.0005)\n")

    def __enter__(self):
        # a separate process polls NVML (~2 kHz), so the samples do not depend on this process's GIL
        try:
            self._p = subprocess.Popen([sys.executable, "-c", self.POLL, str(self.index)], stdout=subprocess.PIPE,
                                       stderr=subprocess.DEVNULL, text=True)
            first = self._p.stdout.readline()  # the poller is running before the timed region starts
            if not first:
                raise RuntimeError("nvml poller failed")
            self._first = first
        except Exception:
            self._p = None
            self._t = threading.Thread(target=self._run_smi, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            out, _ = self._p.communicate(timeout=10)
            for line in (self._first + out).splitlines():
                f = line.split()
                if len(f) == 3:
                    self.rows.append((float(f[0]), float(f[1]), int(f[2])))
        else:
            self._stop.set()
            self._t.join(timeout=10)

    def _run_smi(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout
                for line in out.strip().splitlines():
                    r = [x.strip() for x in line.split(",")]
                    bits = 0
                    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                    for i, n in enumerate(names):
                        if len(r) > 5 + i and r[5 + i] == "Active":
                            bits |= self.BITS[n]
                    if r[1].replace(".", "").isdigit():
                        self.rows.append((float(r[1]), float(r[2]) if r[2].replace(".", "").isdigit() else 0.0, bits))
            except Exception:
                pass
            self._stop.wait(0.2)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for r in self.rows for n, b in self.BITS.items() if r[2] & b})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "sm_mhz_min": min(sm), "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(shape: Shape, target_s: float = 12.0) -> dict:
    """The fp64 oracle as it stands, on all host cores, on a bounded sample of the workload:
    whole (b, h) maps of the workload (fwd + bwd); TFLOP/s from the same flop formula."""
    import oracle
    cores = oracle.default_threads()
    probe = shape.replace(B=1, heads=1)
    inp = make_inputs(probe, seed=1, dtype="bf16", rpb="swin")
    t0 = time.perf_counter()
    oracle.na2d_backward(inp["q"], inp["k"], inp["v"], inp["rpb"], inp["dout"], shape.kernel_size, nthreads=1)
    per_unit = time.perf_counter() - t0
    units = int(max(1, min(shape.units, round(target_s * cores / max(per_unit, 1e-6)))))
    units = max(min(units, shape.units), min(cores, shape.units))
    sample = shape.replace(B=max(1, units // shape.heads), heads=shape.heads if units >= shape.heads else 1)
    inp = make_inputs(sample, seed=2, dtype="bf16", rpb="swin")
    t0 = time.perf_counter()
    oracle.na2d_backward(inp["q"], inp["k"], inp["v"], inp["rpb"], inp["dout"], shape.kernel_size, nthreads=cores)
    dt = time.perf_counter() - t0
    f = sum(flops(sample))
    return {"value": f / dt / 1e12, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{sample.units} (b,h) maps of {shape.name} ({shape.H}x{shape.W}, d={shape.d}, "
                      f"k={shape.kernel_size}), fp64 fwd+bwd, {dt:.2f} s"}


def run_reference(args, shape: Shape):
    """--impl reference: the fp64 oracle (this tier's reference arm), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    cores = oracle.default_threads()
    units = max(1, min(shape.units, 2 * cores))
    sample = shape.replace(B=max(1, units // shape.heads))
    inp = make_inputs(sample, seed=3, dtype="bf16", rpb="swin")

    def step():
        oracle.na2d_backward(inp["q"], inp["k"], inp["v"], inp["rpb"], inp["dout"], shape.kernel_size,
                             nthreads=cores)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = sum(flops(sample)) / dt / 1e12
    desc = (f"{sample.units} (b,h) maps of {shape.name} per step ({shape.H}x{shape.W}, d={shape.d}, "
            f"k={shape.kernel_size}), fp64 fwd+bwd")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(shape, args.gpus, default_mode(shape) if args.mode == "auto" else args.mode),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


MODES = {"weak": "per-rank batch fixed: every rank runs the config's batch (its own batch shard)",
         "units": "fixed problem split by (b, h) units across ranks (heads split when B < ranks)",
         "band": "fixed problem split by query-row bands, (k-1)/2-row K/V halo exchange with the neighbours"}


def default_mode(shape: Shape) -> str:
    """BASELINE configs: NAT-Tiny stages weak-scale by batch; ADE 128^2 is split by batch x heads; the
    COCO map by row bands."""
    if shape.name.startswith("cfg4"):
        return "units"
    if shape.name.startswith("cfg5"):
        return "band"
    return "weak"


def config_dict(shape: Shape, n: int, mode: str = "weak", l2: str | None = None) -> dict:
    par = {"weak": f"dp{n} batch shards, dRPB NCCL all-reduce",
           "units": f"{n} ranks x contiguous (b,h) units, dRPB per-head fold + NCCL all-reduce",
           "band": f"{n} row bands, NCCL send/recv K/V halos + dK/dV halo partials, dRPB all-reduce"}[mode]
    return {"workload": shape.name, "model": "NA2D (NAT-Tiny stage-1 shapes)" if shape.name == DEFAULT_CONFIG else "NA2D",
            "per_rank_batch": shape.B if mode == "weak" else None, "global_batch": shape.B * n if mode == "weak" else shape.B,
            "heads": shape.heads, "H": shape.H, "W": shape.W,
            "head_dim": shape.d, "kernel_size": shape.kernel_size, "rpb": "trunc-normal(0,0.02) table",
            "mode": mode, "parallelism": "single GPU" if n == 1 else par,
            "l2": l2 or "two alternating input sets of 4 x B*heads*H*W*d bf16 (> 126 MB L2 each); no flush"}


def relaunch_distributed(n: int) -> int:
    """`bench.py --gpus N` without a torchrun environment: run this script under torchrun (one rank
    per GPU, rendezvous on 127.0.0.1) and return its exit status."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class Work:
    """One rank's share of a step: inputs resident in HBM, preallocated outputs, step(i)."""

    def __init__(self, args, shape: Shape, mode: str, world: int, rank: int, dev, dist, share: bool):
        import torch
        import paper_2204_07143_b200 as na2d
        from paper_2204_07143_b200 import dist as nd
        self.mode, self.shape, self.world = mode, shape, world
        el = torch.float16 if args.dtype == "f16" else torch.bfloat16
        L, scale = shape.kernel_size, shape.d ** -0.5
        self.L, self.scale = L, scale
        g = shape.replace(B=shape.B * world) if mode == "weak" else shape
        if mode == "weak":
            inp = make_inputs(g, dtype=args.dtype, rpb="swin", batch_offset=rank * shape.B, batch_count=shape.B)
        else:
            inp = make_inputs(g, dtype=args.dtype, rpb="swin")
        full_rpb = torch.from_numpy(inp["rpb"]).to(dev)
        to = lambda x: torch.from_numpy(x).to(dev).to(el)  # noqa: E731
        if mode == "weak":
            t = {n: to(inp[n]) for n in ("q", "k", "v", "dout")}
            self.rpb = full_rpb
        elif mode == "units":
            t = {n: nd.unit_shard(torch.from_numpy(inp[n]), world, rank).to(dev).to(el) for n in ("q", "k", "v", "dout")}
            self.rpb = nd.unit_rpb(full_rpb, shape.B, world, rank)
        else:
            self.band = nd.band_plan(shape.H, world, L)[rank]
            b = self.band
            t = {n: to(np.ascontiguousarray(inp[n][:, :, b.r0:b.r1])) for n in ("q", "dout")}
            for n in ("k", "v"):  # K / V live in the extended band buffer (own rows at [top, top + rows))
                t[n] = to(np.ascontiguousarray(inp[n][:, :, b.k0:b.k1]))
            self.rpb = full_rpb
            self.halo_bufs = [{}, {}]
        del inp
        self.full_rpb = full_rpb
        set_bytes = sum(x.numel() * x.element_size() for x in t.values())
        # L2 hygiene: two alternating input sets when one set exceeds the 126 MB L2, else an L2 flush
        # (256 MB write) before every timed step
        self.flush = None
        if set_bytes >= 150e6:
            self.sets = [t, {n: x.flip(0).contiguous() for n, x in t.items()}]
            self.l2 = f"two alternating input sets of {set_bytes / 1e6:.0f} MB (> 126 MB L2 each); no flush"
        else:
            self.sets = [t]
            self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
            self.l2 = f"input set {set_bytes / 1e6:.1f} MB < L2: 256 MB L2 flush before each step, steps timed one by one"
        q = t["q"]
        self.out = torch.empty_like(q)
        self.lse = torch.empty(q.shape[:4], device=dev, dtype=torch.float32)
        self.dq = torch.empty_like(q)
        self.dk, self.dv = torch.empty_like(t["k"]), torch.empty_like(t["v"])
        self.drpb = torch.empty_like(self.rpb)
        self.drpb_heads = torch.empty_like(full_rpb)
        kw = {}
        if mode == "band":
            kw = dict(map_height=shape.H, q_row0=self.band.r0, kv_row0=self.band.k0)
        self.kw = kw
        self.p = na2d.problem_for(q, t["k"], L, scale, **kw)
        self.ws = torch.empty(max(16, na2d.na2d_backward_workspace_bytes(self.p)), device=dev, dtype=torch.uint8)
        self.nq = q.shape[0] * q.shape[1] * q.shape[2] * q.shape[3]  # this rank's query-heads
        f_fwd, f_bwd = flops(shape)
        self.flops_job = (f_fwd + f_bwd) * (world if mode == "weak" else 1)
        self.dist, self.rank, self.na2d, self.nd = dist, rank, na2d, nd

    def step(self, i):
        na2d, nd, dist = self.na2d, self.nd, self.dist
        s = self.sets[i % len(self.sets)]
        L, scale = self.L, self.scale
        if self.mode == "band":
            nd.exchange_halo(s["k"], self.band, bufs=self.halo_bufs[0])
            nd.exchange_halo(s["v"], self.band, bufs=self.halo_bufs[1])
        na2d.forward(s["q"], s["k"], s["v"], self.rpb, L, scale, out=self.out, lse=self.lse, **self.kw)
        na2d.backward(s["q"], s["k"], s["v"], self.rpb, self.out, self.lse, s["dout"], L, scale, workspace=self.ws,
                      grads=(self.dq, self.dk, self.dv, self.drpb), **self.kw)
        if self.mode == "band":
            if self.world > 1:
                self.dk_own = nd._return_partials(self.dk, self.band).to(self.dk.dtype)
                self.dv_own = nd._return_partials(self.dv, self.band).to(self.dv.dtype)
            nd.allreduce_drpb(self.drpb)
        elif self.mode == "units":
            nd.unit_drpb_to_heads(self.drpb, self.shape.heads, self.shape.B, self.world, self.rank, out=self.drpb_heads)
        elif self.world > 1:
            dist.all_reduce(self.drpb)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS) + sorted(EXTRA_WORKLOADS),
                    help="a BASELINE config (cfg*) or a shape-generality workload (f3_*)")
    ap.add_argument("--mode", default="auto", choices=["auto"] + sorted(MODES),
                    help="multi-GPU partition (auto: the config's; " + "; ".join(f"{k}: {v}" for k, v in MODES.items()) + ")")
    ap.add_argument("--impl", default="na2d", choices=["na2d", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="skip cpu baseline / e2e / clocks (profiling runs)")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f16"],
                    help="16-bit I/O type of the tensor-core path (BASELINE's metric is bf16)")
    args = ap.parse_args()
    shape = CONFIGS[args.config] if args.config in CONFIGS else EXTRA_WORKLOADS[args.config]
    mode = default_mode(shape) if args.mode == "auto" else args.mode

    env_world = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and env_world is None:
        sys.exit(relaunch_distributed(args.gpus))
    if env_world is not None and int(env_world) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, shape)
        return

    import torch
    import torch.distributed as dist
    import paper_2204_07143_b200 as na2d

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test knob: run N ranks on fewer GPUs (ranks share a device, gloo instead of NCCL) to exercise
    # the N > 1 code path on a one-GPU box; never used for reported numbers
    share = os.environ.get("NA2D_BENCH_SHARE_GPU") == "1"
    if share:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    na2d.load_library()
    w = Work(args, shape, mode, world, rank, dev, dist, share)
    p, L, scale = w.p, w.L, w.scale

    def barrier():
        if world > 1:
            dist.barrier() if share else dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    for i in range(args.warmup):
        if w.flush is not None:
            w.flush.fill_(i & 0xff)
        w.step(i)
    barrier()
    sampler = ClockSampler(local) if not args.no_extras else None
    if sampler:
        sampler.__enter__()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    if w.flush is None:
        e0.record()
        for i in range(args.steps):
            w.step(i)
        e1.record()
        barrier()
        ms = e0.elapsed_time(e1) / args.steps
    else:  # steps timed one by one, an untimed L2 flush before each
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            w.flush.fill_(i & 0xff)
            evs[i][0].record()
            w.step(i)
            evs[i][1].record()
        barrier()
        ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    if sampler:
        sampler.__exit__()
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    f_fwd, f_bwd = flops(shape)
    value = w.flops_job / (ms * 1e-3) / 1e12
    launches_per_step = na2d.na2d_launch_count(p, 0) + na2d.na2d_launch_count(p, 1)

    # ---- per-kernel CUDA-event timing (same steps, recorded by the library on its stream)
    na2d.na2d_profile_enable(True)
    for i in range(args.steps):
        if w.flush is not None:
            w.flush.fill_(i & 0xff)
        w.step(i)
    torch.cuda.synchronize()
    prof = na2d.na2d_profile_read()
    na2d.na2d_profile_enable(False)
    peaks = measured_peaks()
    # whole-step algorithmic bytes per query-head: forward 8d + 4 (q, k, v, out, lse),
    # backward 16d + 4 (q, k, v, dout, out, dq, dk, dv, lse): 776 B at d = 32
    step_bytes = (8 * shape.d + 4) + (16 * shape.d + 4)
    kernels = {}
    nq = w.nq
    for name, (tot, cnt) in prof.items():
        per = alg_bytes_per_query(name, shape.d, 2)
        avg_ms = tot / cnt
        kernels[name] = {"avg_us": avg_ms * 1e3, "launches": cnt,
                         "achieved_gbs": (per * nq / (avg_ms * 1e-3) / 1e9) if per else None}
    dom = max(kernels, key=lambda k: kernels[k]["avg_us"] * kernels[k]["launches"]) if kernels else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if dom and os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(shape.name, {}).get(dom)
    roofline = None
    if dom:
        ach = kernels[dom]["achieved_gbs"]
        rank_ms = sum(k["avg_us"] * k["launches"] for k in kernels.values()) / 1e3 / args.steps
        roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": ach / peaks["hbm_gbs"] if ach else None, "traffic": traffic,
                    "alg_bytes_per_launch": alg_bytes_per_query(dom, shape.d, 2) * nq,
                    "peak_source": peaks["_source"], "kernels": kernels,
                    "step_frac_hbm": (step_bytes * nq / (ms * 1e-3) / 1e9) / peaks["hbm_gbs"],
                    "kernels_frac_hbm": (step_bytes * nq / (rank_ms * 1e-3) / 1e9) / peaks["hbm_gbs"],
                    "step_frac_tensor": w.flops_job / world / (ms * 1e-3) / 1e12 / peaks.get("bf16_tflops", 1659.7)}

    # ---- context: the paper's own decomposition (QK+RPB kernel writing the attention
    # weights, softmax, AV, and their gradients) on the same inputs, same device
    paper = None
    if not args.no_extras and args.dtype == "bf16" and mode == "weak" and world == 1:
        s0 = w.sets[0]
        rpb = w.rpb
        _, _, attn = na2d.paper_forward(s0["q"], s0["k"], s0["v"], rpb, L, scale)
        dsb = torch.empty_like(attn)

        def pstep(i):
            s = w.sets[i % len(w.sets)]
            na2d.paper_forward(s["q"], s["k"], s["v"], rpb, L, scale)
            na2d.paper_backward(s["q"], s["k"], s["v"], rpb, attn, s["dout"], L, scale, dS=dsb)

        for i in range(2):
            pstep(i)
        barrier()
        k3 = max(3, min(args.steps, 10))
        e0.record()
        for i in range(k3):
            pstep(i)
        e1.record()
        barrier()
        pms = e0.elapsed_time(e1) / k3
        paper = {"value": (f_fwd + f_bwd) / (pms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": pms,
                 "attn_bytes": attn.numel() * 4, "speedup_fused_vs_paper": pms / ms,
                 "what": "paper's unfused decomposition on this GPU (na2d_paper_forward/backward, CUDA-core kernels)"}
        del attn, dsb

    # ---- end to end through the host-buffer C-ABI entry (pinned host memory); whole maps only
    e2e = None
    if not args.no_extras and mode != "band":
        host = {n: w.sets[0][n].cpu().pin_memory() for n in ("q", "k", "v", "dout")}
        hrpb = w.rpb.cpu().pin_memory()
        hout = {n: torch.empty_like(host["q"]).pin_memory() for n in ("out", "dq", "dk", "dv")}
        hlse = torch.empty(host["q"].shape[:4]).pin_memory()
        hdrpb = torch.empty_like(hrpb).pin_memory()
        nb = na2d.na2d_step_host_workspace_bytes(p)
        w.sets = None
        torch.cuda.empty_cache()
        hws = torch.empty(nb, device=dev, dtype=torch.uint8)
        st = torch.cuda.current_stream().cuda_stream

        def hstep():
            na2d.na2d_step_host(p, host["q"].data_ptr(), host["k"].data_ptr(), host["v"].data_ptr(),
                                hrpb.data_ptr(), host["dout"].data_ptr(), hout["out"].data_ptr(), hlse.data_ptr(),
                                hout["dq"].data_ptr(), hout["dk"].data_ptr(), hout["dv"].data_ptr(),
                                hdrpb.data_ptr(), hws.data_ptr(), nb, st)
            if world > 1:
                d = hdrpb.to(dev)
                if mode == "units":
                    d = w.nd.unit_drpb_to_heads(d, shape.heads, shape.B, world, rank)
                else:
                    dist.all_reduce(d)
                d.cpu()

        hstep()
        barrier()
        k2 = max(3, min(args.steps, 10))
        e0.record()
        for _ in range(k2):
            hstep()
        e1.record()
        barrier()
        ems = e0.elapsed_time(e1) / k2
        if world > 1:
            tt = torch.tensor([ems], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        tb = host["q"].numel() * 2
        TT = hrpb.numel() * 4
        e2e = {"value": w.flops_job / (ems * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": 4 * tb + TT, "d2h_bytes_per_step": 4 * tb + hlse.numel() * 4 + TT,
               "path": "na2d_step_host (pinned host buffers; H2D + fwd + bwd + D2H pipelined over up to 16 batch chunks on three library streams)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_extras:
        cpu = cpu_baseline(shape)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak" if mode == "weak" else "strong",
                "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
                "config": config_dict(shape, world, mode, w.l2),
                "impl": "na2d", "gpu_launches": launches_per_step * args.steps,
                "kernel_families": [na2d.na2d_kernel_family(p, 0), na2d.na2d_kernel_family(p, 1)],
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "paper_design": paper,
                "clocks": sampler.summary() if sampler else None}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
