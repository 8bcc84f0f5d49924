L=$PWD/paper_2012_03119_b200
echo base; timeout 90 python tools/profile_round.py C3 3 2>&1 | tail -1
echo persist; TSG_L2_PERSIST=1 timeout 90 python tools/profile_round.py C3 3 2>&1 | tail -1
echo mb4; TSG_LIB=$L/libtsg_mb4.so timeout 90 python tools/profile_round.py C3 3 2>&1 | tail -1
echo mb4+persist; TSG_L2_PERSIST=1 TSG_LIB=$L/libtsg_mb4.so timeout 90 python tools/profile_round.py C3 3 2>&1 | tail -1
echo C2; timeout 90 python tools/profile_round.py C2 3 2>&1 | tail -1
echo C2 persist; TSG_L2_PERSIST=1 timeout 90 python tools/profile_round.py C2 3 2>&1 | tail -1
timeout 900 python tools/exchange_loop.py 20000 8 60 > gpurun_out/c5.log 2>&1; cat gpurun_out/c5.log
