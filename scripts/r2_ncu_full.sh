# r2: one ncu --set full capture of the step's kernels (after the same command exits 0 without ncu)
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/profile_step.py --steps 4 > gpurun_out/r2e_profile_plain.log 2>&1 && \
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k regex:"sim_tile|grad_gemm|fc_anchor|fc_prep" \
  -s 6 -c 6 -o gpurun_out/r2e_full python scripts/profile_step.py --steps 4 > gpurun_out/r2e_ncu_full.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/r2e_ncu_full.log
