#!/bin/bash
# compute-sanitizer over the round-2 paths (head dims 16 / 64 on tcgen05, SIMT d = 128 with the
# fixed-order dRPB) and the d = 32 kernels; summaries into gpurun_out/sanitizer_r02_*.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py s7 d16 d64 d64k5f16 d128 pair7 pair3 > gpurun_out/sanitizer_r02_$tool.txt 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer_r02_$tool.txt
  tail -3 gpurun_out/sanitizer_r02_$tool.txt
done
