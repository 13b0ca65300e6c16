"""Peer-copy bandwidth between GPU 0 and 1 from one process (copy engine over NVLink)."""
import torch
for mb in (2.6, 10.5, 64):
    n = int(mb * 1e6)
    a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    for _ in range(3): b.copy_(a, non_blocking=True)
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.device(0):
        e0.record()
        for _ in range(20): b.copy_(a, non_blocking=True)
        e1.record()
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    t = e0.elapsed_time(e1) / 20
    print(f"{mb} MB: {t*1e3:.1f} us, {n/t/1e6:.0f} GB/s", flush=True)
# kernel-driven peer stores (SM copy): write into the peer's buffer from a kernel
torch.cuda.set_device(0)
n = int(10.5e6) // 4
src = torch.randn(n, device="cuda:0")
dst = torch.empty(n, device="cuda:1")
for _ in range(3): dst.copy_(src)
torch.cuda.synchronize(0); torch.cuda.synchronize(1)
