# K > 1: parity with the bulk-copy embedding gather, then an A/B of FC_PEER_BULK at N = 2 / 4
mkdir -p gpurun_out/r2m
FC_PEER_BULK=1 timeout -s KILL 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q -k "skewed or ranks_match" 2>&1 | grep -E "^FAILED|passed|failed|^E  " | head
for n in 2 4; do
for rep in 1 2; do
for v in 0 1; do
  FC_PEER_BULK=$v timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29514 \
    bench.py --gpus $n --steps 50 --warmup 5 --no-e2e > gpurun_out/r2m/ab.json 2> gpurun_out/r2m/ab.err
  python -c "import json; d=json.loads(open('gpurun_out/r2m/ab.json').read().strip().splitlines()[-1]); print('N=$n bulk=$v', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})" || tail -3 gpurun_out/r2m/ab.err
done; done; done
