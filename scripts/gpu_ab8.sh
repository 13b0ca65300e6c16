# A/B: anchor-kernel lanes per anchor (8 / 16 / 32), 1 GPU; parity of each build first
for L in 16 32; do
  FC_LIB_PATH=paper_2407_01445_b200/lib/ab_l$L.so timeout -s KILL 300 python -m pytest tests/test_gpu_step.py -q -x --timeout 200 -k "small or ragged or config1" 2>&1 | grep -E "^E |passed|failed" | head -3
done
for i in 1 2 3; do
  for L in 8 16 32; do
    FC_LIB_PATH=paper_2407_01445_b200/lib/ab_l$L.so timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('lanes $L', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d.get('phases_ms',{}).items()})" || tail -2 gpurun_out/ab.err
  done
done
