mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -3
timeout -s KILL 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo "rc=$?"
tail -2 gpurun_out/bench8.err; python -c "import json; d=json.load(open('gpurun_out/bench8.json')); print(d['ms_per_step'], d['step_roofline']['frac'], {k:round(v*1e3,1) for k,v in d['phases_ms'].items()})"
echo "=== multicast"
FC_GEMM_MC=1 timeout -s KILL 120 python -m pytest tests/test_gpu_step.py -q -x --timeout 60 -k "config1 or v3" 2>&1 | tail -3
FC_GEMM_MC=1 timeout -s KILL 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo "rc=$?"
tail -2 gpurun_out/bench9.err; python -c "import json; d=json.load(open('gpurun_out/bench9.json')); print(d['ms_per_step'], d['step_roofline']['frac'], {k:round(v*1e3,1) for k,v in d['phases_ms'].items()})"
