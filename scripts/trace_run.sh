#!/bin/bash
# Build libna2d with the pipeline timeline compiled in (-DNA2D_TRACE) and dump the traces.
NA2D_NVCC_EXTRA="-DNA2D_TRACE ${EXTRA}" python -c "from paper_2204_07143_b200 import build; build.build(force=True)" > gpurun_out/build_trace.log 2>&1 || { tail gpurun_out/build_trace.log; exit 1; }
for s in ${TRACES:-trace_fwd}; do timeout 120 python scripts/$s.py 2>&1 | tee gpurun_out/$s.log | head -40; done
