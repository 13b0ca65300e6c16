import ctypes as C, os, sys, numpy as np, torch
sys.path.insert(0, '.')
os.environ['FC_SIM_DEBUG'] = '9'
os.environ['FC_GRAPH'] = '1'
import paper_2407_01445_b200 as P
from paper_2407_01445_b200 import synthetic as S
B, d, N = 5120, 512, 2_700_000
cfg = P.config_defaults('fastclip_v3', N, dim=d, local_batch=B)
st = P.LossStep(cfg)
b1, b2 = S.embeddings(B, d, 0)
e1 = torch.from_numpy(b1.view(np.int16)).cuda().view(torch.bfloat16)
e2 = torch.from_numpy(b2.view(np.int16)).cuda().view(torch.bfloat16)
ids = torch.from_numpy(S.ids(B, N, 0)).cuda()
for _ in range(3): st.step(e1, e2, ids, 0.6, 1e-14)
torch.cuda.synchronize()
out = np.zeros(2 * 1664, dtype=np.int64)
P.lib().fc_debug_counters(st._h, out.ctypes.data_as(C.POINTER(C.c_longlong)))
for k, name in enumerate(('pass1', 'pass2')):
    reg = out[k * 1664:(k + 1) * 1664]
    o = reg[:1024].reshape(128, 8)[:74]
    tl = reg[1024:].reshape(160, 4)[:148]
    print(name, 'MMA-warp cycles: total', o[:, 0].mean(), 'max', o[:, 0].max(), 'tempty', o[:, 1].mean(), 'afull', o[:, 2].mean(), 'full', o[:, 3].mean(), 'first', o[:, 4].mean())
    e0 = tl[:, 0].min()
    print('   timeline us: entry spread', (tl[:, 0].max() - e0) / 1e3, 'work_end min/max', (tl[:, 1].min() - e0) / 1e3, (tl[:, 1].max() - e0) / 1e3, 'exit max', (tl[:, 2].max() - e0) / 1e3)
for k, name in enumerate(('pass1', 'pass2')):
    reg = out[k * 1664:(k + 1) * 1664]
    e = reg[:1024].reshape(128, 8)[80:80 + 48]
    print(name, 'epilogue warp cycles: total', e[:, 0].mean(), 'wait tfull', e[:, 1].mean(), 'tmem ld', e[:, 2].mean(), 'math', e[:, 3].mean())
for k, name in enumerate(('pass1', 'pass2')):
    reg = out[k * 1664:(k + 1) * 1664]
    tl = reg[1024:].reshape(160, 4)[:148]
    print('zero-entry CTAs', np.nonzero(tl[:, 0] == 0)[0][:10], 'nonzero', (tl[:, 0] != 0).sum())
    tl = tl[(tl[:, 0] > 10**17) & (tl[:, 1] > 10**17)]   # rows 0-25 overlap the epilogue-counter region
    e0 = tl[:, 0].min()
    tl = (tl - e0).astype(np.float64)
    e0 = 0
    ent = np.sort((tl[:, 0] - e0) / 1e3); we = np.sort((tl[:, 1] - e0) / 1e3)
    print(name, 'entry pct', np.round(ent[np.linspace(0, len(ent) - 1, 5).astype(int)], 2), 'work_end pct', np.round(we[np.linspace(0, len(we) - 1, 5).astype(int)], 2))
st.enable_phase_timing(5)
for _ in range(5): st.step(e1, e2, ids, 0.6, 1e-14)
torch.cuda.synchronize()
print('phases (debug9 build)', {k: round(v * 1e3, 1) for k, v in st.phase_times(4).items()})

