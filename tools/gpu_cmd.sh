timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
echo pivot; timeout 120 python tools/profile_round.py C3 3 2>&1 | tail -1
echo nopivot; TSG_PIVOT=0 timeout 120 python tools/profile_round.py C3 3 2>&1 | tail -1
echo C2 pivot; timeout 120 python tools/profile_round.py C2 3 2>&1 | tail -1
echo C2 nopivot; TSG_PIVOT=0 timeout 120 python tools/profile_round.py C2 3 2>&1 | tail -1
