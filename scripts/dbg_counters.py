"""Profiling counters of the step's kernels (diagnostics; results of the step are valid). Needs the
profiling build: FC_PROFILE=1 python -m paper_2407_01445_b200.build --force, then FC_PROF=1."""
import ctypes as C, os, sys, numpy as np, torch
sys.path.insert(0, '.')
os.environ['FC_PROF'] = '1'
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
R = 2688
out = np.zeros(2 * R + 160 * 16 + 8192, dtype=np.int64)
P.lib().fc_debug_counters(st._h, out.ctypes.data_as(C.POINTER(C.c_longlong)))
for k, name in enumerate(('pass1', 'pass2')):
    reg = out[k * R:(k + 1) * R]
    o = reg[:1024].reshape(128, 8)[:74]
    e = reg[1024:2048].reshape(128, 8)[:74]
    tl = reg[2048:].reshape(160, 4)[:148]
    t0 = tl[:, 0].min()
    us = lambda x: np.round(np.percentile((x - t0) / 1e3, [0, 50, 100]), 2)
    print(f'{name}: MMA-warp cycles total {o[:, 0].mean():.0f} (max {o[:, 0].max()}) waits: tempty {o[:, 1].mean():.0f} afull {o[:, 2].mean():.0f} full {o[:, 3].mean():.0f} first-MMA {o[:, 4].mean():.0f}; items {o[:, 6].min()}-{o[:, 6].max()}')
    print(f'   epilogue warp cycles total {e[:, 0].mean():.0f} wait tfull {e[:, 1].mean():.0f} math {e[:, 3].mean():.0f}')
    print('   timeline us [min, median, max] from first CTA entry: entry', us(tl[:, 0]), 'epi start', us(e[:, 4]),
          'MMA end', us(o[:, 7]), 'epi end', us(e[:, 5]), 'work end', us(tl[:, 1]), 'exit', us(tl[:, 2]))
st.enable_phase_timing(5)
for _ in range(5): st.step(e1, e2, ids, 0.6, 1e-14)
torch.cuda.synchronize()
print('phases (debug9 build)', {k: round(v * 1e3, 1) for k, v in st.phase_times(4).items()})
g = out[2 * R:2 * R + 160 * 16].reshape(160, 16)[:148]
if True:
    ld = g[0::2]   # pair leaders (MMA counters)
    t0 = g[:, 11].min()
    us = lambda x: np.round(np.percentile((x - t0) / 1e3, [0, 50, 100]), 2)
    print(f'GEMM: MMA-warp cycles total {ld[:, 0].mean():.0f} (max {ld[:, 0].max()}) waits: tempty {ld[:, 1].mean():.0f} full {ld[:, 2].mean():.0f} first {ld[:, 3].mean():.0f}; units {ld[:, 4].min()}-{ld[:, 4].max()}')
    print(f'   epilogue warp0 cycles total {g[:, 8].mean():.0f} wait tfull {g[:, 9].mean():.0f}')
    print('   timeline us: entry', us(g[:, 11]), 'MMA end', us(ld[:, 5]), 'epi end', us(g[:, 10]))
# absolute step timeline from the per-CTA globaltimer stamps (ns): one graph replay
for _ in range(2): st.step(e1, e2, ids, 0.6, 1e-14)
st.disable_phase_timing()
for _ in range(3): st.step(e1, e2, ids, 0.6, 1e-14)
torch.cuda.synchronize()
out[:] = 0
P.lib().fc_debug_reset(st._h)
st.step(e1, e2, ids, 0.6, 1e-14)
torch.cuda.synchronize()
P.lib().fc_debug_counters(st._h, out.ctypes.data_as(C.POINTER(C.c_longlong)))
tls = [out[k * R + 2048:k * R + 2048 + 148 * 4].reshape(148, 4) for k in range(2)]
g = out[2 * R:2 * R + 160 * 16].reshape(160, 16)[:148]
t0 = tls[0][:, 0].min()
f = lambda x: round((x - t0) / 1e3, 2)
print('graph-step timeline (us from pass-1 first CTA entry):')
print('  pass1: first entry', f(tls[0][:, 0].min()), 'last entry', f(tls[0][:, 0].max()), 'first exit', f(tls[0][:, 2].min()), 'last exit', f(tls[0][:, 2].max()))
print('  pass2: first entry', f(tls[1][:, 0].min()), 'last entry', f(tls[1][:, 0].max()), 'first exit', f(tls[1][:, 2].min()), 'last exit', f(tls[1][:, 2].max()))
if True:
    print('  gemm : first entry', f(g[:, 11].min()), 'last entry', f(g[:, 11].max()), 'epi end min', f(g[:, 10].min()), 'epi end max', f(g[:, 10].max()))
an = out[2 * R + 160 * 16:2 * R + 160 * 16 + 640 * 8].reshape(640, 8)
an = an[an[:, 0] != 0]
pc = lambda x: [f(v) for v in np.percentile(x, [0, 10, 50, 90, 100])]
print(f'  anchor ({len(an)} blocks) [min p10 p50 p90 max]: entry', pc(an[:, 0]), 'wait done', pc(an[:, 1]),
      'partials reduced', pc(an[:, 2]), 'fp64 done', pc(an[:, 3]), 'exit', pc(an[:, 4]))
print('  prep: first entry', f(out[2 * R + 160 * 16 + 8 * 640]), 'last exit', f(out[2 * R + 160 * 16 + 8 * 640 + 1]))
