timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
echo varmajor; timeout 120 python tools/profile_round.py C3 4 2>&1 | tail -1
echo groupmajor; TSG_LANE_GROUP_MAJOR=1 timeout 120 python tools/profile_round.py C3 4 2>&1 | tail -1
echo C2 varmajor; timeout 120 python tools/profile_round.py C2 4 2>&1 | tail -1
echo C2 groupmajor; TSG_LANE_GROUP_MAJOR=1 timeout 120 python tools/profile_round.py C2 4 2>&1 | tail -1
echo int8 varmajor; TSG_INT8_ROWS=1 timeout 120 python tools/profile_round.py C3 4 2>&1 | tail -1
