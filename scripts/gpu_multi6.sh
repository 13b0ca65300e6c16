mkdir -p gpurun_out
nvidia-smi -L | wc -l
for n in 4 2; do
  timeout --kill-after=10 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 30 --warmup 5 > gpurun_out/n$n.out 2> gpurun_out/n$n.err
  echo "N=$n rc=$?"
  tail -1 gpurun_out/n$n.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), d['e2e']['value'], {k:round(v*1e3,1) for k,v in d['phases_ms'].items()})" || grep -a "rror" gpurun_out/n$n.err | head -3
done
