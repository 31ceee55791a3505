#!/bin/bash
# build libna2d variants: build_variants.sh name1 "flags1" name2 "flags2" ... -> paper_2204_07143_b200/_build/libna2d_<name>.so
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  NA2D_NVCC_EXTRA="$2" python -c "from paper_2204_07143_b200 import build as b; b.build(force=True)" || exit 1
  cp paper_2204_07143_b200/libna2d.so paper_2204_07143_b200/_build/libna2d_$1.so
  shift 2
done
python -c "from paper_2204_07143_b200 import build as b; b.build(force=True)"
