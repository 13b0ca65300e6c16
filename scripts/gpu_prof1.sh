set -x
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout -s KILL 200 python scripts/profile_step.py --steps 3 > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:sim_tile_kernel -s 2 -c 2 -o gpurun_out/prof_sim -f python scripts/profile_step.py --steps 3 > gpurun_out/ncu_sim.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:grad_gemm -s 1 -c 1 -o gpurun_out/prof_gemm -f python scripts/profile_step.py --steps 3 > gpurun_out/ncu_gemm.log 2>&1
timeout -s KILL 200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_plain.json 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
