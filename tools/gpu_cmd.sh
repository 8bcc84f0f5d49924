timeout 600 python -m pytest tests/test_gpu_engine.py -m gpu -x -q --timeout 300 -p no:cacheprovider -k "error_paths or async" 2>&1 | tail -15
