run() { env "$@" timeout --kill-after=10 60 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/nccl_probe.py 2>&1 | grep "world" | sed "s/^/[$*] /"; }
run NCCL_DEBUG=WARN
run NCCL_NVLS_ENABLE=0
run NCCL_ALGO=Ring NCCL_NVLS_ENABLE=0
run NCCL_PROTO=Simple NCCL_NVLS_ENABLE=0
run NCCL_PROTO=LL128 NCCL_NVLS_ENABLE=0
run NCCL_MIN_NCHANNELS=32 NCCL_NVLS_ENABLE=0
run NCCL_P2P_USE_CUDA_MEMCPY=1 NCCL_NVLS_ENABLE=0
