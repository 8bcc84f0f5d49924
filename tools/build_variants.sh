#!/bin/bash
# Build k_test variants side by side (libtsg_<tag>.so) for tools/gpu_kprobe.sh.
#   tools/build_variants.sh "tag:-DFLAG=1 ..." ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  tag=${v%%:*}; flags=${v#*:}
  TSG_NVCC_FLAGS="$flags -Xptxas -v" python paper_2012_03119_b200/build.py --force --out=paper_2012_03119_b200/libtsg_$tag.so 2>&1 \
    | grep -A2 "k_testIjjLb0" | grep -E "spill|Used" | tr '\n' ' '; echo " <- $tag"
done
