mkdir -p gpurun_out
timeout -s KILL 200 python scripts/profile_step.py --steps 3 > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"grad_gemm" -s 1 -c 1 -o gpurun_out/prof6 -f python scripts/profile_step.py --steps 3 > gpurun_out/ncu6.log 2>&1
tail -1 gpurun_out/ncu6.log
