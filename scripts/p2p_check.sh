nvidia-smi topo -m 2>&1 | head -8
python -c "import torch; print('can_access_peer 0->1', torch.cuda.can_device_access_peer(0,1))"
NCCL_DEBUG=INFO timeout --kill-after=10 100 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/nccl_probe.py 2>&1 | grep -E "via|Channel 00|NVLS|world|P2P|SHM|transport|NCCL INFO Using|comm 0x" | head -30
