# r2 final evidence, 1 GPU: the -m gpu suite, smoke, the default bench line (with the full CPU
# reference step), the ncu launch list of the same bench command and one ncu --set full capture
# of the step's kernels (each ncu pass only after its command exited 0 without ncu)
set -o pipefail
mkdir -p gpurun_out/r2g
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/r2g/gpu.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 | tee gpurun_out/r2g/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout -s KILL 900 python bench.py > gpurun_out/r2g/bench.json 2> gpurun_out/r2g/bench.err && echo bench ok
cut -c1-400 gpurun_out/r2g/bench.json
timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2g/bench_small.json 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2g_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2g/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout -s KILL 300 python scripts/profile_step.py --steps 4 > gpurun_out/r2g_profile_plain.log 2>&1 && \
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k regex:"sim_tile|grad_gemm|fc_anchor|fc_prep" \
  -s 6 -c 6 -o gpurun_out/r2g_full python scripts/profile_step.py --steps 4 > gpurun_out/r2g_ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/r2g_ncu_full.log
