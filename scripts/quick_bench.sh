#!/bin/bash
# build + one bench line (kernel times only) for fast A/B iterations
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python bench.py --no-extras --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/qb.json 2> gpurun_out/qb.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/qb.json").read().strip().splitlines()[-1])
print("ms/step", round(d["ms_per_step"], 4), "TFLOP/s", round(d["value"], 2))
for k, v in d["roofline"]["kernels"].items():
    print(k, round(v["avg_us"], 1), "us")
PY
for c in ${ONE_CASES}; do timeout 60 python scripts/one_case.py ${c//,/ }; done
