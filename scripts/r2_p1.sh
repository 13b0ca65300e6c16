mkdir -p gpurun_out/r2/configs
timeout -s KILL 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_engine.py tests/test_gpu_fullsize.py -m gpu -q 2>&1 | grep -E "^FAILED|passed|failed|^E  " | head -20
run() {
  local name=$1; shift
  timeout -s KILL 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" > gpurun_out/r2/configs/$name.json 2> gpurun_out/r2/configs/$name.err
  python -c "import json; d=json.load(open('gpurun_out/r2/configs/$name.json')); print('$name', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})" || tail -5 gpurun_out/r2/configs/$name.err
}
run ns_v3
run v3_tau0.01 --tau 0.01
run cfg2_v2_B8192 --variant fastclip_v2 --batch 8192 --n-train 9100000
run v2_B5120 --variant fastclip_v2
