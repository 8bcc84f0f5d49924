# k_test block shapes at 24 warps per SM, built on the box (scratch copy)
for v in "256 3" "192 4" "128 6" "384 2"; do
  set -- $v
  TSG_NVCC_FLAGS="-DTSG_TEST_THREADS=$1 -DTSG_TEST_MIN_BLOCKS=$2" timeout 600 python -c "from paper_2012_03119_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/bv.log 2>&1
  echo "$1x$2 $(tail -1 gpurun_out/bv.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["kernel_ms"])' 2>&1 | tail -1)"
done
