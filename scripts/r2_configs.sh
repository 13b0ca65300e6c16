# r2: throughput lines for the BASELINE.json configs beyond the headline (one GPU each) ->
# gpurun_out/r2/configs/*.json and a markdown table
mkdir -p gpurun_out/r2/configs
timeout -s KILL 600 python -m pytest tests/test_gpu_step.py -m gpu -q -k "latch or config1" 2>&1 | tail -2
run() {   # name, bench args
  local name=$1; shift
  timeout -s KILL 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/r2/configs/$name.json 2> gpurun_out/r2/configs/$name.err
  python -c "import json; d=json.load(open('gpurun_out/r2/configs/$name.json')); print('| $name |', round(d['ms_per_step']*1e3,1), '|', round(d['value'],1), '|', round(d['e2e']['value'],1), '|', round(d['step_roofline']['frac'],3), '|', ' / '.join(str(round(d['phases_ms'][k]*1e3,1)) for k in ('pass1_stats','pass2_q','grad_gemm')), '|')" || tail -5 gpurun_out/r2/configs/$name.err
}
echo "| config | us / step | steps/s | e2e steps/s | step frac of peak | pass 1 / pass 2 / GEMM us |"
echo "|---|---|---|---|---|---|"
run ns_v3_B5120_d512
run v3_tau0.01 --tau 0.01
run cfg1_v3_B256 --batch 256
run cfg2_v2_B8192_N9.1M --variant fastclip_v2 --batch 8192 --n-train 9100000
run v2_B5120 --variant fastclip_v2
run cfg3_v3_d768_N315M --dim 768 --n-train 315000000
run cfg4_v0_B4096_d1024 --variant fastclip_v0 --batch 4096 --dim 1024
run cfg4_v2_B4096_d1024 --variant fastclip_v2 --batch 4096 --dim 1024
run cfg5_v3_B16384 --batch 16384
run cfg5_v3_B32768 --batch 32768
