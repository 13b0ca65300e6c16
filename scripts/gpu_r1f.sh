# r1f: round-end evidence at HEAD on a fresh box (run with gpurun --gpus 2)
mkdir -p gpurun_out/r1f
timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 180 > gpurun_out/r1f/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r1f/pytest_gpu.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1f/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r1f/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r1f/bench_n1.json 2> gpurun_out/r1f/bench_n1.err; echo "bench rc=$?"; cat gpurun_out/r1f/bench_n1.json
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r1f/bench_n2.json 2> gpurun_out/r1f/bench_n2.err; echo "bench2 rc=$?"; tail -c 600 gpurun_out/r1f/bench_n2.json
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1f/bench_ref.json 2> gpurun_out/r1f/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/r1f/bench_ref.json
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1f/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1f/ncu.log 2>&1; echo "ncu rc=$?"
