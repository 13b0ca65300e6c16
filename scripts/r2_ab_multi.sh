# A/B of the K > 1 step: this build vs the round-1 library (FC_LIB_PATH) and without the
# duplicate-id check, N = 4, same box, alternating
mkdir -p gpurun_out/r2m
for rep in 1 2; do
for v in new old nodup; do
  unset FC_LIB_PATH FC_DUP_CHECK
  [ $v = old ] && export FC_LIB_PATH=$PWD/_ab/lib_r1.so
  [ $v = nodup ] && export FC_DUP_CHECK=0
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 4 --steps 50 --warmup 5 --no-e2e > gpurun_out/r2m/ab.json 2> gpurun_out/r2m/ab.err
  python -c "import json; d=json.loads(open('gpurun_out/r2m/ab.json').read().strip().splitlines()[-1]); print('N=4 $v', round(d['ms_per_step']*1e3,1), 'us')" || tail -3 gpurun_out/r2m/ab.err
done
done
