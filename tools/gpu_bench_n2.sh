#!/bin/bash
# The bench's N>1 path on one GPU (every rank on the same device, gloo
# carrying the collectives): strong scaling, split tables, merged records
# verified against the unsharded store.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for mode in ${MODES:-split bcast}; do
TSG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --e2e-steps 3 --tables $mode --verify ${ARGS} > gpurun_out/bench_n2_$mode.log 2>&1
echo "n2 $mode rc=$?"
tail -1 gpurun_out/bench_n2_$mode.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['scaling'], d['value'], d['ms_per_step'], d['config']['clauses_per_gpu'], d['verify'], d['e2e'].get('ms_per_step'), d['config']['parallelism'])" || tail -30 gpurun_out/bench_n2_$mode.log
done
