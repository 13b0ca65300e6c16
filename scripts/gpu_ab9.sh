# A/B: previous build (lib/ab_l8.so) vs current, after the GPU suite; then the step timeline
timeout -s KILL 600 python -m pytest tests/test_gpu_step.py -q -x --timeout 300 2>&1 | grep -E "^E |passed|failed" | head -4
for i in 1 2 3; do
  for lib in ab_l8 libfastclip_b200; do
    FC_LIB_PATH=paper_2407_01445_b200/lib/$lib.so timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$lib', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d.get('phases_ms',{}).items()})" || tail -2 gpurun_out/ab.err
  done
done
timeout -s KILL 300 python scripts/dbg_counters.py 2>&1 | tail -6
