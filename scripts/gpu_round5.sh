mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests -m gpu -q --timeout 120 2>&1 | tail -3
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo "rc=$?"
tail -2 gpurun_out/bench7.err; python -c "import json; d=json.load(open('gpurun_out/bench7.json')); print(d['ms_per_step'], d['value'], d['step_roofline']['frac'], d['e2e']['value'], {k:round(v*1e3,1) for k,v in d['phases_ms'].items()}, d['clocks'])"
timeout -s KILL 120 python scripts/dbg_counters.py 2>&1 | tail -8
