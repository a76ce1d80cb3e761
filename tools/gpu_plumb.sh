# bench.py multi-rank plumbing on one GPU (2 ranks on cuda:0, gloo, host-driven
# slab PCG: a functional check, never a measurement), then the default N=1 bench
mkdir -p gpurun_out/pl
MQ_BENCH_PLUMBING_TEST=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --skip-secondary \
  > gpurun_out/pl/n2.log 2>&1
echo "n2 rc=$?"
grep '^{' gpurun_out/pl/n2.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('n2', d['n_gpus'], d['value'], json.dumps(d['cfg4_sharded'])[:400])"
tail -3 gpurun_out/pl/n2.log
