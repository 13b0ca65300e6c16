# K > 1: parity, then this build vs the previous commit's library at N = 2 / 4 (same box)
mkdir -p gpurun_out/r2m
timeout -s KILL 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q -k "skewed or ranks_match or fallback" 2>&1 | grep -E "^FAILED|passed|failed|^E  " | head
for n in 2 4; do
for rep in 1 2; do
for v in new prev; do
  unset FC_LIB_PATH; [ $v = prev ] && export FC_LIB_PATH=$PWD/_ab/lib_prev.so
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29515 \
    bench.py --gpus $n --steps 50 --warmup 5 --no-e2e > gpurun_out/r2m/ab.json 2> gpurun_out/r2m/ab.err
  python -c "import json; d=json.loads(open('gpurun_out/r2m/ab.json').read().strip().splitlines()[-1]); print('N=$n $v', round(d['ms_per_step']*1e3,1), 'us')" || tail -3 gpurun_out/r2m/ab.err
done; done; done
