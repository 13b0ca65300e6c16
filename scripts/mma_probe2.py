"""tcgen05 issue-rate probe: K-major vs MN-major operands (diagnostics)."""
import ctypes as C, os, sys, torch
sys.path.insert(0, '.')
import paper_2407_01445_b200 as P
L = C.CDLL(os.environ.get('FC_PROBE_LIB', '/tmp/libmma_probe.so'))   # built from paper_2407_01445_b200/probes/mma_probe.cu
L.probe_mma.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
pairs, n_mma = 74, 4096
for name, flags in (("K/K", 1 | 2 | 4), ("A K, B MN", 1 | 2 | 4 | 8), ("A MN, B MN", 1 | 2 | 4 | 8 | 16), ("A MN, B K", 1 | 2 | 4 | 16)):
    cyc = torch.zeros(pairs, dtype=torch.int64, device='cuda')
    s = torch.cuda.current_stream()
    for _ in range(2):
        rc = L.probe_mma(pairs, n_mma, flags, cyc.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    print(f"{name}: {cyc.float().mean().item() / n_mma:.1f} cyc/MMA (ideal 128) rc={rc}", flush=True)
