# r2 round evidence, 1 GPU: the -m gpu suite, the default bench line (with the full CPU
# reference step), and the ncu launch list of the same bench command (exits 0 without ncu first)
set -o pipefail
mkdir -p gpurun_out/r2e
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/r2e/gpu.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 | tee gpurun_out/r2e/pytest_gpu.log
timeout -s KILL 900 python bench.py > gpurun_out/r2e/bench.json 2> gpurun_out/r2e/bench.err && echo bench ok
cut -c1-600 gpurun_out/r2e/bench.json
timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e/bench_small.json 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2e_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e/ncu_launch.log 2>&1; echo "ncu rc=$?"
