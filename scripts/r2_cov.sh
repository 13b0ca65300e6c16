# r2: coverage rows on one GPU (state I/O, model step) + the whole 1-GPU suite
mkdir -p gpurun_out/r2
timeout -s KILL 1200 python -m pytest tests -m gpu -q 2>&1 | grep -E "^FAILED|passed|failed|^E  .*Error" | head -40
