mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests -m gpu -q -x --timeout 150 2>&1 | grep -E "^E |passed|failed" | head -10
timeout --kill-after=10 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/n2.out 2> gpurun_out/n2.err
echo "bench rc=$?"
tail -1 gpurun_out/n2.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'], {k:round(v*1e3,1) for k,v in d['phases_ms'].items()})"
