#!/bin/bash
# One GPU call of evidence: the random-gather microbenchmarks, ncu --set full
# captures of the two hot kernels at C3, and the launch list of the bench
# command itself (ncu --metrics gpu__time_duration.sum, B200_PROFILING.md).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for b in probe gather_modes tma_gather; do
  timeout 300 tools/microbench/$b > gpurun_out/micro_$b.txt 2>&1; echo "$b rc=$?"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_test -s 2 -c 1 -o gpurun_out/${TAG:-r02}_C3_k_test -f \
  python tools/profile_round.py C3 3 > gpurun_out/ncu_test.log 2>&1; echo "ncu k_test rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_encode -s 2 -c 1 -o gpurun_out/${TAG:-r02}_C3_k_encode -f \
  python tools/profile_round.py C3 3 > gpurun_out/ncu_enc.log 2>&1; echo "ncu k_encode rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG:-r02}_launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 3 --no-cpu-baseline --no-api > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ls -la gpurun_out | head -30
