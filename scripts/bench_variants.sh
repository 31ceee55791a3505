#!/bin/bash
# on the GPU box: time each prebuilt variant (bench.py --no-extras), print per-kernel us
cd "$(dirname "$0")/.."
cp paper_2204_07143_b200/libna2d.so /tmp/libna2d_main.so
for v in "$@"; do
  cp paper_2204_07143_b200/_build/libna2d_$v.so paper_2204_07143_b200/libna2d.so
  for rep in 1 2; do
    python bench.py --steps 20 --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step']*1000,1), {k:round(v['avg_us'],1) for k,v in d['roofline']['kernels'].items()})"
  done
done
cp /tmp/libna2d_main.so paper_2204_07143_b200/libna2d.so
