# A/B: GEMM B-operand multicast (clusters of 2 pairs, persistent grid) vs pairs, 1 GPU
FC_GEMM_MC=1 timeout -s KILL 500 python -m pytest tests/test_gpu_step.py -q -x --timeout 300 2>&1 | grep -E "^E |passed|failed" | head -4
for i in 1 2 3; do
  for cfg in "FC_GEMM_MC=1" "FC_GEMM_MC=0"; do
    env $cfg timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$cfg', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d.get('phases_ms',{}).items()})" || tail -2 gpurun_out/ab.err
  done
done
