#!/bin/bash
# Pipeline traces of forward experiment variants (-DNA2D_TRACE -DNA2D_EXP=k)
for k in ${EXPS:-0 2 4}; do
  NA2D_NVCC_EXTRA="-DNA2D_TRACE -DNA2D_EXP=$k" python -c "from paper_2204_07143_b200 import build; build.build(force=True)" > gpurun_out/build_texp$k.log 2>&1 || { tail -5 gpurun_out/build_texp$k.log; continue; }
  echo "EXP=$k"; timeout 120 python scripts/trace_fwd.py 2>&1 | grep "tile  9" -A0
done
