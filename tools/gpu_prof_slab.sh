#!/bin/bash
# ncu capture of the slab kernel at C3 (one launch) + source page
ncu --set full --clock-control none --import-source on -k regex:k_test_slab -s 1 -c 1 -o gpurun_out/prof_slab python tools/profile_round.py C3 2 > gpurun_out/ncu_slab.log 2>&1
tail -3 gpurun_out/ncu_slab.log
