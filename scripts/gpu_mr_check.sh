timeout -s KILL 600 python -m pytest tests/test_gpu_multirank.py -q -x --timeout 300 2>&1 | grep -E "^E |passed|failed" | head -5
bash scripts/gpu_mr_timeline.sh | grep "rep 2"
bash scripts/gpu_multi10.sh
