#!/bin/bash
# GPU-box check: the GPU test suite, then a short bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^ERROR|^E  " gpurun_out/pytest_gpu.log | head -30
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench.log 2>&1
  echo "bench rc=$?"
  tail -1 gpurun_out/bench.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['roofline']['encode_ms'], d['e2e'].get('ms_per_step'))" || tail -20 gpurun_out/bench.log
fi
