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

from na2d_inputs import CONFIGS, Shape, make_inputs  # noqa: E402

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
            "config": config_dict(shape, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(shape: Shape, n: int) -> dict:
    return {"workload": shape.name, "model": "NA2D (NAT-Tiny stage-1 shapes)" if shape.name == DEFAULT_CONFIG else "NA2D",
            "per_rank_batch": shape.B, "global_batch": shape.B * n, "heads": shape.heads, "H": shape.H, "W": shape.W,
            "head_dim": shape.d, "kernel_size": shape.kernel_size, "rpb": "trunc-normal(0,0.02) table",
            "parallelism": f"dp{n} batch shards, dRPB NCCL all-reduce" if n > 1 else "single GPU",
            "l2": "two alternating input sets of 4 x B*heads*H*W*d bf16 (> 126 MB L2 each); no flush"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="na2d", choices=["na2d", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="skip cpu baseline / e2e / clocks (profiling runs)")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f16"],
                    help="16-bit I/O type of the tensor-core path (BASELINE's metric is bf16)")
    args = ap.parse_args()
    shape = CONFIGS[args.config]
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

    # ---- inputs: this rank's batch shard of the global synthetic batch, resident in HBM
    g = shape.replace(B=shape.B * world)
    inp = make_inputs(g, dtype=args.dtype, rpb="swin", batch_offset=rank * shape.B, batch_count=shape.B)
    el = torch.float16 if args.dtype == "f16" else torch.bfloat16
    sets = []
    t = {n: torch.from_numpy(inp[n]).to(dev).to(el) for n in ("q", "k", "v", "dout")}
    sets.append(t)
    sets.append({n: x.flip(0).contiguous() for n, x in t.items()})
    rpb = torch.from_numpy(inp["rpb"]).to(dev)
    del inp
    L, scale = shape.kernel_size, shape.d ** -0.5
    out = torch.empty_like(t["q"])
    lse = torch.empty(t["q"].shape[:4], device=dev, dtype=torch.float32)
    dq, dk, dv = torch.empty_like(out), torch.empty_like(out), torch.empty_like(out)
    drpb = torch.empty_like(rpb)
    p = na2d.problem_for(t["q"], t["k"], L, scale)
    ws = torch.empty(max(16, na2d.na2d_backward_workspace_bytes(p)), device=dev, dtype=torch.uint8)

    def step(i):
        s = sets[i % 2]
        na2d.forward(s["q"], s["k"], s["v"], rpb, L, scale, out=out, lse=lse)
        na2d.backward(s["q"], s["k"], s["v"], rpb, out, lse, s["dout"], L, scale, workspace=ws,
                      grads=(dq, dk, dv, drpb))
        if world > 1:
            dist.all_reduce(drpb)

    def barrier():
        if world > 1:
            dist.barrier() if share else dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    for i in range(args.warmup):
        step(i)
    barrier()
    sampler = ClockSampler(local) if not args.no_extras else None
    if sampler:
        sampler.__enter__()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    for i in range(args.steps):
        step(i)
    e1.record()
    barrier()
    if sampler:
        sampler.__exit__()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    f_fwd, f_bwd = flops(shape)
    value = (f_fwd + f_bwd) * world / (ms * 1e-3) / 1e12
    launches_per_step = na2d.na2d_launch_count(p, 0) + na2d.na2d_launch_count(p, 1)

    # ---- per-kernel CUDA-event timing (same steps, recorded by the library on its stream)
    na2d.na2d_profile_enable(True)
    for i in range(args.steps):
        step(i)
    torch.cuda.synchronize()
    prof = na2d.na2d_profile_read()
    na2d.na2d_profile_enable(False)
    peaks = measured_peaks()
    kernels = {}
    nq = shape.units * shape.H * shape.W
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
        roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": ach / peaks["hbm_gbs"] if ach else None, "traffic": traffic,
                    "alg_bytes_per_launch": alg_bytes_per_query(dom, shape.d, 2) * nq,
                    "peak_source": peaks["_source"], "kernels": kernels,
                    "step_frac_hbm": ((260 + 516) * nq / (ms * 1e-3) / 1e9) / peaks["hbm_gbs"],
                    "step_frac_tensor": (f_fwd + f_bwd) / (ms * 1e-3) / 1e12 / peaks.get("bf16_tflops", 1659.7)}

    # ---- context: the paper's own decomposition (QK+RPB kernel writing the attention
    # weights, softmax, AV, and their gradients) on the same inputs, same device
    paper = None
    if not args.no_extras and args.dtype == "bf16":  # the comparison path has no fp16 I/O
        s0 = sets[0]
        _, _, attn = na2d.paper_forward(s0["q"], s0["k"], s0["v"], rpb, L, scale)
        dsb = torch.empty_like(attn)

        def pstep(i):
            s = sets[i % 2]
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

    # ---- end to end through the host-buffer C-ABI entry (pinned host memory)
    e2e = None
    if not args.no_extras:
        host = {n: sets[0][n].cpu().pin_memory() for n in ("q", "k", "v", "dout")}
        hrpb = rpb.cpu().pin_memory()
        hout = {n: torch.empty_like(host["q"]).pin_memory() for n in ("out", "dq", "dk", "dv")}
        hlse = torch.empty(host["q"].shape[:4]).pin_memory()
        hdrpb = torch.empty_like(hrpb).pin_memory()
        nb = na2d.na2d_step_host_workspace_bytes(p)
        del sets
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
                dist.all_reduce(d)
                hdrpb.copy_(d)

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
        TT = (2 * L - 1) ** 2 * shape.heads * 4
        e2e = {"value": (f_fwd + f_bwd) * world / (ems * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": 4 * tb + TT, "d2h_bytes_per_step": 4 * tb + hlse.numel() * 4 + TT,
               "path": "na2d_step_host (pinned host buffers; H2D + fwd + bwd + D2H pipelined over up to 16 batch chunks on three library streams)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_extras:
        cpu = cpu_baseline(shape)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": args.dtype, "data": "synthetic", "config": config_dict(shape, world),
                "impl": "na2d", "gpu_launches": launches_per_step * args.steps,
                "kernel_families": [na2d.na2d_kernel_family(p, 0), na2d.na2d_kernel_family(p, 1)],
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "paper_design": paper,
                "clocks": sampler.summary() if sampler else None}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
