#!/bin/bash
# One GPU-box session: build, tests, smoke, bench, ncu launch list (+ optional full capture).
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -z "${SKIP_TESTS}" ]; then
  timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
if [ -n "${NCU}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/ncu_bench.log 2>&1
fi
if [ -n "${NCU_FULL}" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${NCU_FULL}" -s 1 -c 1 -o gpurun_out/prof_full python scripts/prof_fwd.py cfg2_nat_tiny_s1 3 --bwd > gpurun_out/ncu_full.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log 2>/dev/null; cat gpurun_out/bench.json
