set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
mkdir -p gpurun_out
timeout -s KILL 240 python -m pytest tests/test_gpu_step.py -x -q -k similarity 2>&1 | tail -20
timeout -s KILL 400 python -m pytest tests/test_gpu_step.py -x -q 2>&1 | tail -40
