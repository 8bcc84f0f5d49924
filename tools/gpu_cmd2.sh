TSG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-ingress split > gpurun_out/bench_n2.log 2>&1; tail -1 gpurun_out/bench_n2.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['e2e'])[:900])"
grep -i "error\|Traceback" gpurun_out/bench_n2.log | head -5
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench1.log 2>&1; tail -1 gpurun_out/bench1.log | cut -c1-200
