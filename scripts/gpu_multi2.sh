mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_multirank.py -q -x --timeout 150 2>&1 | grep -E "^E |assert|Error|passed|failed" | head -20
timeout -s KILL 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench rc=$?"
grep -v "^frame\|^\[rank\|^Exception\|^$" gpurun_out/bench_n2.err | tail -5
python -c "import json; d=json.load(open('gpurun_out/bench_n2.json')); print(d['ms_per_step'], {k:round(v*1e3,1) for k,v in d['phases_ms'].items()})"
