# 4 GPUs: profiled single-step timelines, chunked embedding gather on / off (same build)
export FC_PEER_TIMEOUT_MS=5000 FC_LIB_PATH=$PWD/_ab/lib_prof.so
for c in 1 0; do
  echo "== chunks=$c"
  FC_GATHER_CHUNKS=$c timeout -s KILL 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 \
    scripts/dbg_timeline_mr.py 2>&1 | grep -E "^rank 0" | sed 's/np.float64(\([^)]*\))/\1/g' | cut -c1-330
done
