# 4 GPUs: multicast embedding gather -- is it on, multi-rank parity, steps / bench vs _ab/lib_prev.so
export FC_PEER_TIMEOUT_MS=3000
FC_MC_VERBOSE=1 timeout -s KILL 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29516 \
    scripts/dbg_steps_mr.py 2>&1 | grep -E "multicast|^rank 0|Error" | head -5
timeout -s KILL 600 python -m pytest tests/test_gpu_multirank.py -m gpu -q -x 2>&1 | grep -E "passed|failed|Error|assert" | head -6
for v in new prev; do
  unset FC_LIB_PATH; [ $v = prev ] && export FC_LIB_PATH=$PWD/_ab/lib_prev.so
  timeout -s KILL 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29516 \
    scripts/dbg_steps_mr.py 2>&1 | grep "^rank 0" | sed "s/^/$v /"
done
