#!/bin/bash
# one gpurun call: GPU tests (short summary), then the bench line; outputs under gpurun_out/
tag=${1:-x}
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/gputest_$tag.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
tail -3 gpurun_out/gputest_$tag.txt
python -c "
import json; d=json.loads(open('gpurun_out/bench_$tag.json').read().strip().splitlines()[-1])
print('ms/step', d['ms_per_step'], 'TFLOP/s', d['value']); print({k:round(v['avg_us'],1) for k,v in d['roofline']['kernels'].items()})"
