mkdir -p gpurun_out
nvidia-smi -L
timeout -s KILL 400 python -m pytest tests/test_gpu_multirank.py -q -x --timeout 300 2>&1 | tail -5
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_n2.err; cat gpurun_out/bench_n2.json | head -c 400; echo
