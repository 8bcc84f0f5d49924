for v in 0 1 0 1; do
TSG_DYN_TILES=$v timeout 600 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench$v.log 2>&1
tail -1 gpurun_out/bench$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print($v, d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['encode_ms'], d['roofline'].get('l2_gather'))"
done
