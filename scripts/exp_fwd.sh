#!/bin/bash
# Forward timing experiments: build libna2d variants with -DNA2D_EXP=k, time the forward in bench.py
for k in ${EXPS:-0 1 2 3}; do
  NA2D_NVCC_EXTRA="-DNA2D_EXP=$k" python -c "from paper_2204_07143_b200 import build; build.build(force=True)" > gpurun_out/build_exp$k.log 2>&1 || { tail -5 gpurun_out/build_exp$k.log; continue; }
  echo -n "EXP=$k "; timeout 120 python bench.py --steps 10 --warmup 3 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:round(v['avg_us'],1) for k,v in d['roofline']['kernels'].items()})"
done
