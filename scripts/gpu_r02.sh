#!/bin/bash
# Round-2 GPU session: build, gpu tests, smoke, bench (cfg2), launch list, ncu --set full per kernel.
#   TAG=vN KERNELS="na2d_fwd_tc na2d_bwd_dq na2d_bwd_dkdv" SKIP_TESTS= bash scripts/gpu_r02.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-v0}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -z "${SKIP_TESTS}" ]; then
  NA2D_PARITY_LOG=gpurun_out/r02_parity_errors_$TAG.jsonl timeout 1200 python -m pytest tests -m gpu -q -x -rs > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
  tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -3 gpurun_out/smoke_$TAG.log
fi
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench exit $?"
cut -c1-1500 gpurun_out/bench_$TAG.json
if [ -z "${SKIP_NCU}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-extras ${BENCH_ARGS} > gpurun_out/ncu_bench_$TAG.log 2>&1
  python scripts/launch_shares.py gpurun_out/launches_$TAG.csv
fi
for k in ${KERNELS}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" -s 2 -c 1 -o gpurun_out/full_${TAG}_$k -f \
    python scripts/prof_fwd.py ${PROF_CFG:-cfg2_nat_tiny_s1} 4 --bwd > gpurun_out/ncu_${TAG}_$k.log 2>&1
  echo "ncu $k exit $?"
done
if [ -n "${KERNELS}" ]; then
  python scripts/ncu_summary.py gpurun_out/ncu_full_$TAG.md ${PROF_CFG:-cfg2_nat_tiny_s1} gpurun_out/full_${TAG}_*.ncu-rep
fi
