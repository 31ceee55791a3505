#!/bin/bash
# Timing experiments over compile-flag variants: FLAGSETS="-DA=1;-DB=2" (';'-separated), each built
# with NA2D_NVCC_EXTRA, checked by PYTEST_K (optional) and timed per kernel with bench.py.
IFS=';' read -ra SETS <<< "${FLAGSETS}"
i=0
for f in "${SETS[@]}"; do
  i=$((i+1))
  NA2D_NVCC_EXTRA="$f" python -c "from paper_2204_07143_b200 import build; build.build(force=True)" > gpurun_out/build_fs$i.log 2>&1 || { echo "[$f] build failed"; tail -5 gpurun_out/build_fs$i.log; continue; }
  if [ -n "${PYTEST_K}" ]; then timeout 300 python -m pytest tests -m gpu -q -x -k "${PYTEST_K}" 2>&1 | tail -1; fi
  for r in 1 2; do
  echo -n "[$f] "; timeout 120 python bench.py --steps 20 --warmup 5 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), {k:round(v['avg_us'],1) for k,v in d['roofline']['kernels'].items()})"
  done
done
