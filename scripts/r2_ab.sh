# same-box A/B of an env switch on the default bench step (alternating); usage: AB="FC_X=0 FC_X=1" bash scripts/r2_ab.sh
mkdir -p gpurun_out/r2
for rep in 1 2; do
  for v in $AB; do
    env $v timeout -s KILL 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2/ab.json 2>gpurun_out/r2/ab.err
    python -c "import json,sys; d=json.load(open('gpurun_out/r2/ab.json')); print('$v', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})" || tail -3 gpurun_out/r2/ab.err
  done
done
