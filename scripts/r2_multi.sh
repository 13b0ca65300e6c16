# r2: multi-GPU evidence on one box (N = 2 / 4): K > 1 parity incl. the rank-skew stress test,
# then the bench line at N = 2 and N = 4 (torchrun, one rank per GPU)
mkdir -p gpurun_out/r2m
N=$(nvidia-smi -L | wc -l)
timeout -s KILL 1800 python -m pytest tests/test_gpu_multirank.py -m gpu -q -s 2>&1 | grep -E "worst|passed|failed|^FAILED|^E  " | head -30 | tee gpurun_out/r2m/pytest_multirank.log
for n in 2 4; do
  [ "$n" -le "$N" ] || continue
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r2m/bench_n$n.json 2> gpurun_out/r2m/bench_n$n.err
  python -c "import json; d=json.load(open('gpurun_out/r2m/bench_n$n.json')); print('N=$n', round(d['ms_per_step']*1e3,1), 'us', round(d['value'],1), 'steps/s e2e', round(d['e2e']['value'],1), {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})" || tail -5 gpurun_out/r2m/bench_n$n.err
done
