mkdir -p gpurun_out
export FC_BENCH_TRACE=1
timeout --kill-after=10 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/n2.out 2> gpurun_out/n2.err
echo "bench rc=$?"
grep -a "bench rank\|rror\|Traceback" gpurun_out/n2.err | grep -v TCPStore | tail -4
python -c "import json; d=json.load(open('gpurun_out/n2.out')); print(d['ms_per_step'], d['e2e'], {k:round(v*1e3,1) for k,v in d['phases_ms'].items()})"
cat > /tmp/close_test.py <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import torch.multiprocessing as mp
def w(rank, nid, q):
    import paper_2407_01445_b200 as P
    torch.cuda.set_device(rank)
    cfg = P.config_defaults("fastclip_v3", 4096, dim=128, local_batch=256, world=2, rank=rank, device=rank)
    for i, b in enumerate(nid): cfg.nccl_id[i] = b
    st = P.LossStep(cfg)
    e = torch.randn(256, 128, device=f"cuda:{rank}").to(torch.bfloat16)
    ids = torch.arange(256, dtype=torch.int32, device=f"cuda:{rank}") + 256 * rank
    for k in range(4): st.step(e, e, ids, 0.6, 1e-14)
    st.enable_phase_timing(2)
    for k in range(2): st.step(e, e, ids, 0.6, 1e-14)
    st.disable_phase_timing()
    torch.cuda.synchronize()
    st.close()
    q.put(rank)
if __name__ == "__main__":
    import paper_2407_01445_b200 as P
    nid = P.nccl_unique_id()
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    ps = [ctx.Process(target=w, args=(r, nid, q)) for r in range(2)]
    [p.start() for p in ps]
    print("closed ranks", sorted(q.get(timeout=100) for _ in range(2)), flush=True)
    [p.join(30) for p in ps]
    print("exitcodes", [p.exitcode for p in ps], flush=True)
PY

