#!/bin/bash
# Profiling session: build, gpu tests + smoke, pipeline traces, ncu --set full of each NA2D kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -z "${SKIP_TESTS}" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
  tail -3 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log
fi
for s in ${TRACES}; do timeout 120 python scripts/$s.py > gpurun_out/$s.log 2>&1; done
for k in ${KERNELS}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" -s 2 -c 1 -o gpurun_out/full_$k -f \
    python scripts/prof_fwd.py cfg2_nat_tiny_s1 4 --bwd > gpurun_out/ncu_$k.log 2>&1
  echo "ncu $k exit $?"
done
