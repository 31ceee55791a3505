#!/bin/bash
# on the GPU box: per-kernel times (bench.py --no-extras) for the given configs with each prebuilt
# library variant: ab_configs.sh "cfg2_nat_tiny_s1 cfg4_ade20k_128" variant1 variant2 ...
# (variant "main" = the in-tree libna2d.so)
cd "$(dirname "$0")/.."
cfgs=$1; shift
cp paper_2204_07143_b200/libna2d.so paper_2204_07143_b200/_build/libna2d_main.so
for rep in 1 2; do
  for v in "$@"; do
    cp paper_2204_07143_b200/_build/libna2d_$v.so paper_2204_07143_b200/libna2d.so
    for c in $cfgs; do
      python bench.py --config $c --steps 20 --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$c', round(d['ms_per_step']*1000,1), {k:round(v['avg_us'],1) for k,v in d['roofline']['kernels'].items()})"
    done
  done
done
cp paper_2204_07143_b200/_build/libna2d_main.so paper_2204_07143_b200/libna2d.so
