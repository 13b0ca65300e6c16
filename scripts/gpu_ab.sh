# A/B of env switches on the bench step time (graph replay), alternating runs
mkdir -p gpurun_out
for i in 1 2; do
  for v in "FC_FUSED_P1=1" "FC_FUSED_P1=0"; do
    env $v timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print('$v', round(d['ms_per_step']*1e3,1), 'us')"
  done
done
