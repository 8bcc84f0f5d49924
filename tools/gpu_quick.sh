#!/bin/bash
# quick GPU check: parity tests, then C3/C2 device-round timing of every built libtsg variant
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for lib in paper_2012_03119_b200/libtsg*.so; do
  echo "== $lib"
  TSG_LIB=$PWD/$lib timeout 300 python tools/profile_round.py C3 3 2>&1 | tail -1
  TSG_LIB=$PWD/$lib TSG_SLABS=0 timeout 300 python tools/profile_round.py C3 3 2>&1 | tail -1
  TSG_LIB=$PWD/$lib timeout 300 python tools/profile_round.py C2 3 2>&1 | tail -1
done
