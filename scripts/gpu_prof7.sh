mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -2
timeout -s KILL 200 python scripts/dbg_counters.py 2>&1 | grep -A2 "^pass1\|phases"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"sim_tile_kernel" -s 2 -c 1 -o gpurun_out/prof7 -f python scripts/profile_step.py --steps 3 > gpurun_out/ncu7.log 2>&1
tail -1 gpurun_out/ncu7.log
