for i in 1 2 3; do
for N in 4 2; do
  timeout --kill-after=10 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/mb.json 2> gpurun_out/mb.err
  tail -1 gpurun_out/mb.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N', round(d['ms_per_step']*1e3,1))"
done
done
