#!/bin/bash
# Round-2 evidence session: tests (+ parity margins), smoke, default bench line, launch list, ncu --set full
# of each kernel at cfg2, then every BASELINE config at N=1 and the N=2 shared-GPU partition paths.
cd "$(dirname "$0")/.."
TAG=${TAG:-final} KERNELS="na2d_fwd_tc na2d_bwd_dq na2d_bwd_dkdv" bash scripts/gpu_r02.sh
bash scripts/bench_configs.sh
