#!/bin/bash
# time every built libtsg variant on C3 and C2 (device-resident rounds)
for lib in paper_2012_03119_b200/libtsg*.so; do
  echo "== $lib"
  TSG_LIB=$PWD/$lib timeout 300 python tools/profile_round.py C3 3 2>&1 | tail -1
done
