timeout 700 python -m pytest tests/test_gpu_engine.py tests/test_gpu_bitpack.py -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 120 python tools/profile_round.py C3 4 2>&1 | tail -1; done
timeout 120 python tools/profile_round.py C2 4 2>&1 | tail -1
