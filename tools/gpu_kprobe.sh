#!/bin/bash
# k_test variants side by side: event timings per library (TSG_LIB), then one
# ncu --set full capture of k_test per library given in NCU_LIBS.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in ${LIBS:-paper_2012_03119_b200/libtsg.so}; do
  echo "== $lib"
  TSG_LIB=$lib timeout 300 python tools/profile_round.py ${CFG:-C3} ${ROUNDS:-8} 2>&1 | tail -4
done
for lib in ${NCU_LIBS}; do
  tag=$(basename $lib .so)
  TSG_LIB=$lib timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_test --launch-skip 2 --launch-count 1 \
     -o gpurun_out/${TAG:-r02}_${tag}_k_test -f python tools/profile_round.py ${CFG:-C3} 3 > gpurun_out/ncu_${tag}.log 2>&1
  echo "ncu $tag rc=$?"
done
