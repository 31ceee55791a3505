#!/bin/bash
# e2e (host-buffer step) timing over compile-flag variants: FLAGSETS="-DA=1;-DB=2"
IFS=';' read -ra SETS <<< "${FLAGSETS}"
for f in "${SETS[@]}"; do
  NA2D_NVCC_EXTRA="$f" python -c "from paper_2204_07143_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "[$f] build failed"; continue; }
  for r in 1 2; do
    echo -n "[$f] "; timeout 300 python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],3))"
  done
done
