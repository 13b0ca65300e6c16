# stream-K drain-cost sweep (FC_GEMM_DRAIN, k-blocks per unit boundary), 1 GPU
for i in 1 2; do
  for dr in 4 8 12 16 24; do
    FC_GEMM_DRAIN=$dr timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('drain $dr', round(d['ms_per_step']*1e3,1), round(d['phases_ms']['grad_gemm']*1e3,1))" || tail -2 gpurun_out/ab.err
  done
done
