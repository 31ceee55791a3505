"""Workload-level benchmark: a full NAT forward (and forward+backward) at
224x224 with random weights, every NA step in libna2d.so.  Prints one JSON line: images/s, the
NA kernels' share of the forward (library CUDA-event profile), and the analytic MACs.

    python scripts/bench_nat.py [--variant tiny] [--batch 128] [--res 224] [--steps 20] [--warmup 5]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_07143_b200 as na2d  # noqa: E402
from paper_2204_07143_b200.nat import NAT, nat_macs  # noqa: E402


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="tiny")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--res", type=int, default=224)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    torch.manual_seed(0)
    dev = torch.device("cuda")
    model = NAT(args.variant, device=dev).eval()
    x = torch.randn(args.batch, 3, args.res, args.res, device=dev, dtype=torch.bfloat16)

    def fwd():
        with torch.no_grad():
            return model(x)

    ms_fwd = timed(fwd, args.steps, args.warmup)

    # NA share of the forward: the library's per-kernel CUDA events over the same forwards
    na2d.na2d_profile_enable(True)
    for _ in range(args.steps):
        fwd()
    torch.cuda.synchronize()
    prof = na2d.na2d_profile_read()
    na2d.na2d_profile_enable(False)
    na_ms = sum(t for t, _ in prof.values()) / args.steps

    # the same forward replayed as one CUDA graph (host launch overhead removed)
    ms_graph = None
    if not args.no_graph:
        try:
            sx = torch.cuda.Stream()
            sx.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(sx):
                fwd()
            torch.cuda.current_stream().wait_stream(sx)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fwd()
            ms_graph = timed(g.replay, args.steps, args.warmup)
        except Exception as exc:  # capture unsupported by some step: report, do not fail
            ms_graph = f"capture failed: {exc}"

    model.train()

    def train_step():
        model.zero_grad(set_to_none=True)
        model(x).float().logsumexp(-1).mean().backward()

    ms_train = timed(train_step, max(3, args.steps // 2), args.warmup)
    macs = nat_macs(args.variant, (args.res, args.res))
    out = {
        "metric": f"NAT-{args.variant} images/s ({args.res}x{args.res}, bf16, random weights)",
        "batch": args.batch,
        "fwd_imgs_per_s": args.batch / (ms_fwd * 1e-3),
        "fwd_ms": ms_fwd,
        "fwd_graph_ms": ms_graph,
        "fwd_graph_imgs_per_s": args.batch / (ms_graph * 1e-3) if isinstance(ms_graph, float) else None,
        "train_fwd_bwd_ms": ms_train,
        "train_imgs_per_s": args.batch / (ms_train * 1e-3),
        "na_kernels_ms_per_fwd": na_ms,
        "na_share_of_fwd": na_ms / ms_fwd,
        "na_kernels": {k: {"ms_per_fwd": t / args.steps, "launches_per_fwd": c / args.steps} for k, (t, c) in prof.items()},
        "gmacs_per_img": {k: v / 1e9 for k, v in macs.items()},
        "fwd_tflops_mac2": 2 * macs["total"] * args.batch / (ms_fwd * 1e-3) / 1e12,
        "data": "synthetic",
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
