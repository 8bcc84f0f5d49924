timeout 700 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for lib in paper_2012_03119_b200/libtsg*.so; do echo "== $lib"; for i in 1 2; do TSG_LIB=$PWD/$lib timeout 120 python tools/profile_round.py C3 4 2>&1 | tail -1; done; TSG_LIB=$PWD/$lib timeout 120 python tools/profile_round.py C2 4 2>&1 | tail -1; done
