# Round evidence: bench line, ncu launch list of the bench command, ncu --set full of the hot kernels
# usage: bash scripts/gpu_profiles.sh <tag>   (then: python scripts/summarize_profiles.py <tag>)
T=${1:-r1c}
mkdir -p gpurun_out
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"sim_tile|grad_gemm|fc_prep|fc_anchor|fc_zero" \
  -s 7 -c 6 -o gpurun_out/${T}_full -f python scripts/profile_step.py --steps 3 > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/${T}_ncu_full.log
