"""Pinned host -> device copy bandwidth at the e2e step's size (10.5 MB) and larger."""
import torch
dev = torch.device("cuda:0")
for mb in (5.24, 10.5, 64, 256):
    n = int(mb * 1e6)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        d.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"H2D {mb:7.2f} MB: {ms*1e3:8.1f} us  {n/ms/1e6:6.1f} GB/s")
