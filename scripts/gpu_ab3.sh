for i in 1 2; do
  for lib in ab_old.so libfastclip_b200.so; do
    FC_LIB_PATH=$PWD/paper_2407_01445_b200/lib/$lib timeout --kill-after=10 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e > gpurun_out/n2.out 2> gpurun_out/n2.err
    tail -1 gpurun_out/n2.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib N=2', round(d['ms_per_step']*1e3,1))"
  done
done
