#!/bin/bash
# one GPU call: parity tests, bench, device-round timing, ncu of both hot kernels, launch list
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout 120 python tools/profile_round.py C3 3 > gpurun_out/prof_plain.log 2>&1; tail -1 gpurun_out/prof_plain.log
timeout 120 python tools/profile_round.py C2 3 > gpurun_out/prof_c2.log 2>&1; tail -1 gpurun_out/prof_c2.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_test -s 1 -c 1 -o gpurun_out/prof_test python tools/profile_round.py C3 2 > gpurun_out/ncu_test.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_encode -s 1 -c 1 -o gpurun_out/prof_encode python tools/profile_round.py C3 2 > gpurun_out/ncu_enc.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_test|k_encode" --csv --log-file gpurun_out/launches.csv python tools/profile_round.py C3 3 > gpurun_out/ncu_launch.log 2>&1
ls gpurun_out
