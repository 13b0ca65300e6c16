import ctypes as C, os, sys, torch
sys.path.insert(0, '.')
import paper_2407_01445_b200 as P
L = C.CDLL(os.environ.get('FC_PROBE_LIB', '/tmp/libmma_probe.so'))   # built from paper_2407_01445_b200/probes/mma_probe.cu
for pairs in (74,):
    for tile_kb, epi in ((8, 1), (8, 8), (8, 16)):
        n_kb = 800
        cyc = torch.zeros(pairs, dtype=torch.int64, device='cuda')
        s = torch.cuda.current_stream()
        rc = L.probe_ring(pairs, n_kb, tile_kb, epi, C.c_void_p(cyc.data_ptr()), C.c_void_p(s.cuda_stream))
        torch.cuda.synchronize()
        c = cyc.float().mean().item()
        print(f"ring pairs={pairs} tile_kb={tile_kb} epi_warps={epi}: {c/(4*n_kb):.1f} cyc/MMA (ideal 128) rc={rc}", flush=True)
