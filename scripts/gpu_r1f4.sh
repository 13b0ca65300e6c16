# r1f: 4-GPU multirank parity tests + N=4 bench at HEAD (run with gpurun --gpus 4)
mkdir -p gpurun_out/r1f
timeout -s KILL 600 python -m pytest tests/test_gpu_multirank.py -m gpu -q --timeout 180 > gpurun_out/r1f/pytest_multirank4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r1f/pytest_multirank4.log
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r1f/bench_n4.json 2> gpurun_out/r1f/bench_n4.err; echo "bench4 rc=$?"; tail -c 400 gpurun_out/r1f/bench_n4.json
