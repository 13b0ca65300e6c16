# A/B: current build vs lib/ab_old.so (previous commit), interleaved, 1 GPU
timeout -s KILL 500 python -m pytest tests/test_gpu_step.py -q -x --timeout 300 2>&1 | grep -E "^E |passed|failed" | head -4
for i in 1 2 3; do
  for lib in paper_2407_01445_b200/lib/ab_old.so paper_2407_01445_b200/lib/libfastclip_b200.so; do
    FC_LIB_PATH=$lib timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$lib', round(d['ms_per_step']*1e3,1))" || tail -2 gpurun_out/ab.err
  done
done
