# 2 GPUs: step distributions and bench lines, this build vs _ab/lib_prev.so (alternating, 2 reps)
export FC_PEER_TIMEOUT_MS=3000
for rep in 1 2; do
for v in new prev; do
  unset FC_LIB_PATH; [ $v = prev ] && export FC_LIB_PATH=$PWD/_ab/lib_prev.so
  timeout -s KILL 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 \
    scripts/dbg_steps_mr.py 2>&1 | grep "^rank 0" | sed "s/^/$v /"
  timeout -s KILL 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 \
    bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench N=2 $v', round(d['ms_per_step']*1e3,1), 'us')"
done; done
