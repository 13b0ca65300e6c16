# r1i: config 5 sweep (v3, d = 512, global B 4k..64k) at N = 1 and N = 4 (run with gpurun --gpus 4)
mkdir -p gpurun_out/r1i
for B in 4096 8192 16384 32768 65536; do
  CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r1i/n1_B$B.json 2> gpurun_out/r1i/n1_B$B.err; echo "N=1 B=$B rc=$?"
done
for B in 16384 65536; do
  timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 4 --batch $B --steps 10 --warmup 3 > gpurun_out/r1i/n4_B$B.json 2> gpurun_out/r1i/n4_B$B.err; echo "N=4 B=$B rc=$?"
done
