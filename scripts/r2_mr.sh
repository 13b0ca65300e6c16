# r2: K>1 parity incl. the rank-skew stress test and the abort test (2 GPUs)
mkdir -p gpurun_out/r2
timeout -s KILL 1500 python -m pytest tests/test_gpu_multirank.py -m gpu -q -s 2>&1 | grep -E "worst|passed|failed|Error|assert" | head -40
