# N-GPU parity (2 ranks) + bench lines at N = 2 and (if present) N = 4
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l); echo "gpus=$NG"
timeout -s KILL 400 python -m pytest tests/test_gpu_multirank.py -q -x --timeout 300 2>&1 | grep -E "^E |passed|failed" | head -5
for N in 2 4; do
  [ $N -gt $NG ] && continue
  timeout --kill-after=10 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 50 --warmup 5 > gpurun_out/r1d_bench_n$N.json 2> gpurun_out/r1d_bench_n$N.err
  echo "N=$N rc=$?"
  tail -1 gpurun_out/r1d_bench_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N', round(d['ms_per_step']*1e3,1), d['value'], d['e2e']['value'], {k:round(v*1e3,1) for k,v in d['phases_ms'].items()})"
done
