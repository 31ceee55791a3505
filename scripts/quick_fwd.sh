#!/bin/bash
# quick GPU iteration: build, forward parity check, forward/backward kernel timings
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python scripts/fwd_check.py ${CHECK_ARGS} > gpurun_out/fwd_check.log 2>&1; echo "exit $?" >> gpurun_out/fwd_check.log
cut -c1-160 gpurun_out/fwd_check.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_quick.json').read().strip().splitlines()[-1]); print('value', round(d['value'],2), 'ms', round(d['ms_per_step'],3)); print({k:(round(v['avg_us'],1), v['achieved_gbs'] and round(v['achieved_gbs'])) for k,v in d['roofline']['kernels'].items()})" || tail -5 gpurun_out/bench_quick.err
