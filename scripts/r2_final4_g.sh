# r2 final evidence, 4 GPUs: the multi-rank parity suite, bench lines at N = 2 and 4
set -o pipefail
mkdir -p gpurun_out/r2g
export FC_PEER_TIMEOUT_MS=5000
timeout -s KILL 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q 2>&1 | tail -3 | tee gpurun_out/r2g/pytest_multirank4.log
for n in 2 4; do
  timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29515 \
    bench.py --gpus $n > gpurun_out/r2g/bench_n$n.json 2> gpurun_out/r2g/bench_n$n.err; echo "N=$n rc=$?"
  cut -c1-300 gpurun_out/r2g/bench_n$n.json
done
