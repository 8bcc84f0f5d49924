for lib in paper_2012_03119_b200/libtsg*.so; do echo "== $lib"; for i in 1 2; do TSG_LIB=$PWD/$lib timeout 120 python tools/profile_round.py C3 4 2>&1 | tail -1 | cut -c1-110; done; done
