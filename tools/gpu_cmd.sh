timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
grep -E "^FAILED|^E " gpurun_out/pytest_gpu.log | head -5
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['roofline']['encode_ms'], d['e2e']['ms_per_step'], d['e2e']['mode'])"
