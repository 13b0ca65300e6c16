# Round-1 evidence: bench line, ncu launch list of the bench command, ncu --set full of the hot kernels
mkdir -p gpurun_out
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r1b_bench.json 2> gpurun_out/r1b_bench.err; echo "bench rc=$?"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r1b_ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"sim_tile|grad_gemm|fc_prep|fc_anchor|fc_zero" \
  -s 7 -c 6 -o gpurun_out/r1b_full -f python scripts/profile_step.py --steps 3 > gpurun_out/r1b_ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/r1b_ncu_full.log
