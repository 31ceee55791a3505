#!/bin/bash
# every BASELINE config at N=1 (bench line each) + the N=2 partition paths with two ranks sharing the GPU
cd "$(dirname "$0")/.."
out=gpurun_out/r02_configs.jsonl
: > $out
for c in cfg2_nat_tiny_s1 cfg1_8x8_k3 cfg3_nat_tiny_s2 cfg3_nat_tiny_s3 cfg3_nat_tiny_s4 cfg4_ade20k_128 cfg5_coco_200x336; do
  python bench.py --config $c --steps 20 --warmup 5 ${EXTRA} 2>gpurun_out/bench_$c.err | tail -1 >> $out
done
NA2D_BENCH_SHARE_GPU=1 python bench.py --gpus 2 --config cfg5_coco_200x336 --steps 5 --warmup 3 --no-extras 2>gpurun_out/share5.err | tail -1 > gpurun_out/r02_share2_cfg5.json
NA2D_BENCH_SHARE_GPU=1 python bench.py --gpus 2 --config cfg4_ade20k_128 --steps 5 --warmup 3 --no-extras 2>gpurun_out/share4.err | tail -1 > gpurun_out/r02_share2_cfg4.json
python -c "
import json
for l in open('$out'):
    d=json.loads(l); print(d['config']['workload'], round(d['ms_per_step'],4), 'ms', round(d['value'],2), 'TFLOP/s', 'frac', round(d['roofline']['frac'],3), 'step_hbm', round(d['roofline']['step_frac_hbm'],3))
"
cat gpurun_out/r02_share2_cfg5.json | cut -c1-300; cat gpurun_out/r02_share2_cfg4.json | cut -c1-300
