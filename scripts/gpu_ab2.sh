mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests -m gpu -q -x --timeout 150 2>&1 | grep -E "^E |passed|failed" | head -5
for i in 1 2; do
  for v in "FC_PDL=1" "FC_PDL=0"; do
    env $v timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print('$v', round(d['ms_per_step']*1e3,1), 'us')" || tail -3 gpurun_out/ab.err
  done
done
