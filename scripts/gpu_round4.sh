mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests -m gpu -q --timeout 120 2>&1 | tail -4
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo "rc=$?"
tail -2 gpurun_out/bench6.err; python -c "import json; d=json.load(open('gpurun_out/bench6.json')); print(d['ms_per_step'], d['value'], d['step_roofline']['frac'], d['e2e']['value'], {k:round(v*1e3,1) for k,v in d['phases_ms'].items()})"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo "ncu rc=$?"
