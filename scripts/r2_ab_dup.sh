mkdir -p gpurun_out/r2
for v in "FC_DUP_CHECK=1" "FC_DUP_CHECK=0" "FC_DUP_CHECK=1" "FC_DUP_CHECK=0"; do
  env $v timeout -s KILL 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2/ab.json 2>gpurun_out/r2/ab.err
  python -c "import json,sys; d=json.load(open('gpurun_out/r2/ab.json')); print('$v', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})"
done
