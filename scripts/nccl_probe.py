"""All-gather timing probe (diagnostics): the step's E all-gather shape through torch's NCCL
process group, eager and CUDA-graph captured; device time per call, max over ranks."""
import os, sys, torch, torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
B, d = 5120, 512
Bl = B // world
x = torch.randn(Bl, d, device="cuda").to(torch.bfloat16)
out = torch.empty(B, d, device="cuda", dtype=torch.bfloat16)
small = torch.randn(7 * Bl + 120, device="cuda", dtype=torch.float64)
sout = torch.empty(world * small.numel(), device="cuda", dtype=torch.float64)
s = torch.cuda.Stream()
def run(fn, n=50):
    for _ in range(5): fn()
    torch.cuda.synchronize(); dist.barrier()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / n * 1e3], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()
ag = lambda: (dist.all_gather_into_tensor(out, x), dist.all_gather_into_tensor(out, x))
sg = lambda: dist.all_gather_into_tensor(sout, small)
r1 = run(ag); r2 = run(sg)
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    for _ in range(3): ag()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        ag()
r3 = run(lambda: g.replay())
if rank == 0:
    print(f"world {world}: E all-gather x2 (2 x {Bl*d*2/1e6:.2f} MB per rank) eager {r1:.1f} us, graph {r3:.1f} us; payload gather ({small.numel()*8/1e3:.0f} KB) {r2:.1f} us", flush=True)
dist.barrier()
dist.destroy_process_group()
