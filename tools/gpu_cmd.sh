timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -x -q --timeout 300 -p no:cacheprovider -k "packed or c1 or widths or c3_full" > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 120 python tools/profile_round.py C3 4 2>&1 | tail -1; done
timeout 120 python tools/profile_round.py C2 4 2>&1 | tail -1
