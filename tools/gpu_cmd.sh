timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -x -q --timeout 600 -k "full_size" -p no:cacheprovider --durations=3 > gpurun_out/pytest_gpu.log 2>&1
tail -6 gpurun_out/pytest_gpu.log
