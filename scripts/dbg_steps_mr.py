"""Per-step device times of back-to-back K > 1 steps (L2 flush between steps, as bench.py), per
rank: quantiles and the slow steps. Launch: torchrun --nproc-per-node K scripts/dbg_steps_mr.py"""
import os, sys, numpy as np, torch
import torch.distributed as tdist
sys.path.insert(0, '.')
import paper_2407_01445_b200 as P
from paper_2407_01445_b200 import synthetic as S
rank, K = int(os.environ['RANK']), int(os.environ['WORLD_SIZE'])
torch.cuda.set_device(rank)
tdist.init_process_group('nccl', device_id=torch.device('cuda', rank))
obj = [P.nccl_unique_id() if rank == 0 else None]
tdist.broadcast_object_list(obj, src=0)
B, d, N = 5120, 512, 2_700_000
Bl = B // K
cfg = P.config_defaults('fastclip_v3', N, dim=d, local_batch=Bl, world=K, rank=rank, device=rank)
for i, b in enumerate(obj[0]): cfg.nccl_id[i] = b
st = P.LossStep(cfg)
lo = rank * Bl
sets = []
for k in range(int(os.environ.get('SETS', '1'))):   # distinct input buffers (one graph each, as bench.py)
    b1, b2 = S.embeddings(B, d, k)
    sets.append((torch.from_numpy(b1[lo:lo + Bl].view(np.int16).copy()).cuda().view(torch.bfloat16),
                 torch.from_numpy(b2[lo:lo + Bl].view(np.int16).copy()).cuda().view(torch.bfloat16),
                 torch.from_numpy(S.ids(B, N, k)[lo:lo + Bl]).cuda()))
smi = None
if os.environ.get('SMI'):   # bench.py's clock sampler running beside the timed steps
    import subprocess
    smi = subprocess.Popen(['nvidia-smi', '-i', str(rank), '--query-gpu=clocks.sm', '--format=csv', '-lms', '200'],
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
n = int(os.environ.get('STEPS', '100'))
for i in range(5): st.step(*sets[i % len(sets)], 0.6, 1e-14)
torch.cuda.synchronize(); tdist.barrier()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
for i in range(n):
    flush.zero_()
    ev[i][0].record(); st.step(*sets[i % len(sets)], 0.6, 1e-14); ev[i][1].record()
torch.cuda.synchronize()
t = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
q = np.percentile(t, [0, 10, 50, 90, 100]).round(1)
slow = [(i, round(x, 1)) for i, x in enumerate(t) if x > 2 * np.median(t)]
print(f'rank {rank}: us min/p10/p50/p90/max {list(q)} mean {t.mean():.1f} slow {slow[:12]}', flush=True)
tdist.barrier()
if smi: smi.terminate()
st.close()
tdist.destroy_process_group()
