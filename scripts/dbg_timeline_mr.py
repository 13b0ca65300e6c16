"""Per-rank step timeline of the K > 1 path (profiling-build globaltimer stamps (FC_PROFILE=1 build, FC_PROF=1), one graph
replay per rank). Launch: torchrun --nproc-per-node K scripts/dbg_timeline_mr.py"""
import ctypes as C, os, sys, numpy as np, torch
import torch.distributed as tdist
sys.path.insert(0, '.')
os.environ['FC_PROF'] = '1'
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
b1, b2 = S.embeddings(B, d, 0)
lo = rank * Bl
e1 = torch.from_numpy(b1[lo:lo + Bl].view(np.int16).copy()).cuda().view(torch.bfloat16)
e2 = torch.from_numpy(b2[lo:lo + Bl].view(np.int16).copy()).cuda().view(torch.bfloat16)
ids = torch.from_numpy(S.ids(B, N, 0)[lo:lo + Bl]).cuda()
for _ in range(5): st.step(e1, e2, ids, 0.6, 1e-14)
torch.cuda.synchronize()
R = 2688
out = np.zeros(2 * R + 160 * 16 + 8192, dtype=np.int64)
lines = []
for rep in range(3):
    tdist.barrier()
    out[:] = 0
    P.lib().fc_debug_reset(st._h)
    st.step(e1, e2, ids, 0.6, 1e-14)
    torch.cuda.synchronize()
    P.lib().fc_debug_counters(st._h, out.ctypes.data_as(C.POINTER(C.c_longlong)))
    tls = [out[k * R + 2048:k * R + 2048 + 148 * 4].reshape(148, 4) for k in range(2)]
    g = out[2 * R:2 * R + 160 * 16].reshape(160, 16)[:148]
    an = out[2 * R + 160 * 16:2 * R + 160 * 16 + 640 * 8].reshape(640, 8)
    an = an[an[:, 0] != 0]
    prep = out[2 * R + 160 * 16 + 8 * 640: 2 * R + 160 * 16 + 8 * 640 + 2]
    t0 = prep[0]
    f = lambda x: round((float(x) - t0) / 1e3, 1)
    ge = g[:, 11][g[:, 11] != 0]
    pe = out[2 * R + 160 * 16 + 6000: 2 * R + 160 * 16 + 6008]
    lines.append(f'rank {rank} rep {rep} (us from prep entry): prep exit {f(prep[1])} | pass1 {f(tls[0][:, 0].min())}..{f(tls[0][:, 2].max())} '
                 f'| gatherE {[f(x) for x in pe[:4]]} | anchor {f(an[:, 0].min())} wait {f(an[:, 1].min())} exit {f(an[:, 4].max())} '
                 f'| gatherP {[f(x) for x in pe[4:]]} | pass2 {f(tls[1][:, 0].min())}..{f(tls[1][:, 2].max())} | gemm {f(ge.min())}..{f(g[:, 10].max())}')
    if rep == 2:   # pass-1 MMA-warp counters per pair (cycles -> us at 1.9 GHz)
        m = out[:74 * 8].reshape(74, 8).astype(np.float64)
        c = lambda x: np.round(x / 1900.0, 1)
        lines.append(f'rank {rank} pass1 pairs: items min/max {int(m[:, 6].min())}/{int(m[:, 6].max())} | loop us mean/max {c(m[:, 0].mean())}/{c(m[:, 0].max())} '
                     f'| wait B mean/max {c(m[:, 3].mean())}/{c(m[:, 3].max())} | wait A {c(m[:, 2].mean())}/{c(m[:, 2].max())} '
                     f'| wait tmem {c(m[:, 1].mean())}/{c(m[:, 1].max())} | first mma {c(m[:, 4].mean())}/{c(m[:, 4].max())} '
                     f'| cta entry {f(tls[0][:, 0].min())}..{f(tls[0][:, 0].max())} work end {f(tls[0][:, 1].min())}..{f(tls[0][:, 1].max())}')
print('\n'.join(lines), flush=True)
tdist.barrier()
st.close()
tdist.destroy_process_group()
