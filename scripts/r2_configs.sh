# r2: throughput lines for the BASELINE.json configs beyond the headline (one GPU each)
mkdir -p gpurun_out/r2/configs
run() {   # name, bench args
  local name=$1; shift
  timeout -s KILL 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/r2/configs/$name.json 2> gpurun_out/r2/configs/$name.err
  python -c "import json; d=json.load(open('gpurun_out/r2/configs/$name.json')); print('$name', round(d['ms_per_step']*1e3,1), 'us', round(d['value'],1), 'steps/s', 'e2e', round(d['e2e']['value'],1), 'step_frac', round(d['step_roofline']['frac'],3), {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})" || tail -5 gpurun_out/r2/configs/$name.err
}
run ns_v3_B5120_d512
run v3_tau0.01 --tau 0.01
run cfg2_v2_B8192 --variant fastclip_v2 --batch 8192 --n-train 9100000
run cfg3_v3_d768_N315M --dim 768 --n-train 315000000
run cfg4_v0_B4096_d1024 --variant fastclip_v0 --batch 4096 --dim 1024
run cfg4_v2_B4096_d1024 --variant fastclip_v2 --batch 4096 --dim 1024
