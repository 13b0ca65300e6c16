NG=$(nvidia-smi -L | wc -l)
for N in 2 4; do
  [ $N -gt $NG ] && continue
  timeout --kill-after=10 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 scripts/dbg_timeline_mr.py 2>&1 | grep "rank .* rep" | sort
done
