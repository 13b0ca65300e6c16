mkdir -p gpurun_out/r2
timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2/bench.json 2>gpurun_out/r2/bench.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench.json')); print(round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})" || tail -20 gpurun_out/r2/bench.err
timeout -s KILL 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_engine.py -m gpu -q 2>&1 | grep -E "AssertionError|passed|failed" | head -30
