timeout 400 python -m pytest tests -m gpu -x -q --timeout 120 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
L=$PWD/paper_2012_03119_b200
for lib in libtsg.so libtsg_c2.so libtsg_c4.so; do
for sb in 110000 135168; do
echo "$lib slab $sb"; TSG_LIB=$L/$lib TSG_SLAB_BYTES=$sb timeout 90 python tools/profile_round.py C3 3 2>&1 | tail -1
done; done
