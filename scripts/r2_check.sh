# r2: 1-GPU parity + bench line (+ phases)
mkdir -p gpurun_out/r2
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not multirank" 2>&1 | tail -15
timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2/bench.json 2>gpurun_out/r2/bench.err
python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench.json')); print(round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})" || tail -20 gpurun_out/r2/bench.err
