timeout -s KILL 300 python -m pytest tests -m gpu -q -x --timeout 150 2>&1 | tail -1
for v in 4 8 12 16 20; do
  FC_GEMM_DRAIN=$v timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('drain $v', round(d['ms_per_step']*1e3,1), round(d['phases_ms']['grad_gemm']*1e3,1))"
done
