# K > 1 embedding-gather / pass-1 overlap: the whole GPU suite (1-4 GPUs), then bench lines of this
# build vs the previous commit's library (_ab/lib_prev.so) at N = 2 / 4
mkdir -p gpurun_out/r2o
export FC_PEER_TIMEOUT_MS=10000
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for n in 2 4; do
for rep in 1 2; do
for v in new prev; do
  unset FC_LIB_PATH; [ $v = prev ] && export FC_LIB_PATH=$PWD/_ab/lib_prev.so
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29515 \
    bench.py --gpus $n --steps 50 --warmup 5 --no-e2e > gpurun_out/r2o/ab.json 2> gpurun_out/r2o/ab_${n}_${v}.err
  python -c "import json; d=json.loads(open('gpurun_out/r2o/ab.json').read().strip().splitlines()[-1]); print('bench N=$n $v', round(d['ms_per_step']*1e3,1), 'us')" || grep -E "Error|error|FC_ERR" gpurun_out/r2o/ab_${n}_${v}.err | head -5
done; done; done
