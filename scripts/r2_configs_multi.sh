# r2: multi-GPU throughput lines (4-GPU box): config 2's per-GPU shape (v2, 1024 anchors per GPU,
# N = 9.1M) at K = 2 / 4, and v2 / v3 at the north-star global batch -> gpurun_out/r2/configs_multi
mkdir -p gpurun_out/r2/configs_multi
export FC_PEER_TIMEOUT_MS=5000
run() {   # name, gpus, bench args
  local name=$1 n=$2; shift 2
  timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29515 \
    bench.py --gpus $n --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" > gpurun_out/r2/configs_multi/$name.json 2> gpurun_out/r2/configs_multi/$name.err
  python -c "import json; d=json.loads(open('gpurun_out/r2/configs_multi/$name.json').read().strip().splitlines()[-1]); print('| $name | $n |', round(d['ms_per_step']*1e3,1), '|', round(d['value'],1), '|', round(d['step_roofline']['frac'],3), '|')" || tail -3 gpurun_out/r2/configs_multi/$name.err
}
echo "| config | GPUs | us / step | steps/s | step frac of peak |"
echo "|---|---|---|---|---|"
run cfg2shape_v2_B2048_N9.1M 2 --variant fastclip_v2 --batch 2048 --n-train 9100000
run cfg2shape_v2_B4096_N9.1M 4 --variant fastclip_v2 --batch 4096 --n-train 9100000
run v2_B5120 2 --variant fastclip_v2
run v2_B5120 4 --variant fastclip_v2
run v3_B5120_tau0.01 2 --tau 0.01
run v3_B5120_tau0.01 4 --tau 0.01
