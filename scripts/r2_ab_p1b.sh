# r2: pass-1 epilogue cost: FC_SIM_DEBUG=1 skips the epilogue math (MMA + TMEM loads only)
mkdir -p gpurun_out/r2a
for v in "FC_FUSED_P1=1 FC_SIM_DEBUG=0" "FC_FUSED_P1=1 FC_SIM_DEBUG=1" "FC_FUSED_P1=0 FC_SIM_DEBUG=0" "FC_FUSED_P1=0 FC_SIM_DEBUG=1" "FC_FUSED_P1=0 FC_SIM_DEBUG=2"; do
  env $v timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2a/ab.json 2>gpurun_out/r2a/ab.err
  python -c "import json,sys; d=json.load(open('gpurun_out/r2a/ab.json')); print('$v', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})"
done
