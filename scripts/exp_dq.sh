#!/bin/bash
# B1 timing experiments: build variants of libna2d with -DNA2D_EXP=k and time B1 (trace_dq.py)
for k in ${EXPS:-1 2 0}; do
  NA2D_NVCC_EXTRA="-DNA2D_EXP=$k" python -c "from paper_2204_07143_b200 import build; build.build(force=True)" > gpurun_out/build_exp$k.log 2>&1
  echo "EXP=$k"; timeout 120 python scripts/trace_dq.py 2>&1 | grep -E "^t 3|cold=False"
done
