#!/bin/bash
# End-of-round-2 evidence: tests (+ parity margins), smoke, default bench line, launch list, ncu --set
# full per kernel, every BASELINE config, f3 shapes, sanitizers (memcheck / racecheck / synccheck).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-v5} KERNELS="na2d_fwd_tc na2d_bwd_dq na2d_bwd_dkdv" bash scripts/gpu_r02.sh
bash scripts/bench_configs.sh
: > gpurun_out/r02_f3.jsonl
for c in f3_d16_s1 f3_d64_s1; do
  python bench.py --config $c --steps 10 --warmup 3 --no-extras 2>/dev/null | tail -1 >> gpurun_out/r02_f3.jsonl
done
bash scripts/sanitize_r02.sh
