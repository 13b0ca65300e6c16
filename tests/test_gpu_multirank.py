"""Multi-GPU parity (K = 2 and 4 ranks, one process per GPU): every rank runs the B200 step on
its contiguous slice of the global batch (trainer.cpp:231-241) and the rank outputs must equal
the K-rank oracle replay of trainer.cpp:427-589 on the whole batch -- the gathered-embedding
rows of dE, the all-reduced G_tau and tau update, the exact batch loss and, for the
individual-temperature variants, the replicated IndividualTemp tables. Needs >= K GPUs
(`gpurun --gpus 2` / `--gpus 4`); skipped otherwise."""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_2407_01445_b200 import synthetic as S

pytestmark = pytest.mark.gpu

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, K, variant, B, d, N, steps, nccl_id, q):
    import torch
    import paper_2407_01445_b200 as P
    from gpu_helpers import gpu_cfg, to_dev_bf16
    try:
        torch.cuda.set_device(rank)
        ocfg = O.default_config(variant, N)
        Bl = B // K
        cfg = gpu_cfg(ocfg, d, Bl, world=K, rank=rank, device=rank)
        for i, b in enumerate(nccl_id):
            cfg.nccl_id[i] = b
        step = P.LossStep(cfg)
        step.load_tables(u1=S.warm_u(N, 0), u2=S.warm_u(N, 1))
        out = []
        lo = rank * Bl
        for s in range(steps):
            b1, b2 = S.embeddings(B, d, 77 + s)
            ids = S.ids(B, N, 77 + s)
            de1, de2 = step.step(to_dev_bf16(b1[lo:lo + Bl], f"cuda:{rank}"), to_dev_bf16(b2[lo:lo + Bl], f"cuda:{rank}"),
                                 torch.from_numpy(ids[lo:lo + Bl]).to(f"cuda:{rank}"), 0.6, 1e-14)
            sc = step.scalars()
            out.append(dict(dE1=de1.cpu().numpy().astype(np.float64), dE2=de2.cpu().numpy().astype(np.float64),
                            loss=sc.loss, gtau=sc.gtau, tau=sc.tau))
        tabs = step.tables()
        step.close()   # communicator teardown before the process exits
        q.put((rank, out, {k: np.asarray(v) for k, v in tabs.items()}, None))
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        q.put((rank, None, None, repr(e)))


def _run(K, variant, B, d, N, steps):
    import torch
    import torch.multiprocessing as mp
    import paper_2407_01445_b200 as P
    if torch.cuda.device_count() < K:
        pytest.skip(f"needs {K} GPUs")
    nccl_id = P.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, K, variant, B, d, N, steps, nccl_id, q)) for r in range(K)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(K):
        rank, out, tabs, err = q.get(timeout=300)
        assert err is None, f"rank {rank}: {err}"
        res[rank] = (out, tabs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # oracle: K-rank replay on the whole batch
    ocfg = O.default_config(variant, N)
    st = O.new_state(ocfg)
    st.u1[:] = S.warm_u(N, 0)
    st.u2[:] = S.warm_u(N, 1)
    refs = []
    for s in range(steps):
        b1, b2 = S.embeddings(B, d, 77 + s)
        ids = S.ids(B, N, 77 + s)
        refs.append(O.step(ocfg, st, K, S.bf16_to_f32(b1).astype(np.float64), S.bf16_to_f32(b2).astype(np.float64),
                           ids, 0.6, 1e-14))
    return res, refs, st


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def _norm_rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("K,variant", [(2, "fastclip_v3"), (2, "fastclip_v2"), (2, "fastclip_v1"),
                                       (4, "fastclip_v3"), (4, "fastclip_v2"), (4, "fastclip_v0")])
def test_ranks_match_oracle(K, variant):
    B, d, N, steps = 1024 if K == 4 else 512, 128, 8192, 2
    res, refs, st = _run(K, variant, B, d, N, steps)
    Bl = B // K
    for s in range(steps):
        ref = refs[s]
        for r in range(K):
            got = res[r][0][s]
            lo = r * Bl
            assert _norm_rel(got["dE1"], ref["dE1"][lo:lo + Bl]) < 2e-3, (variant, s, r, "dE1")
            assert _norm_rel(got["dE2"], ref["dE2"][lo:lo + Bl]) < 2e-3, (variant, s, r, "dE2")
            assert _rel(got["loss"], ref["loss"]) < 1e-3, (variant, s, r, "loss")
            assert _rel(got["tau"], ref["tau_new"]) < 1e-3, (variant, s, r, "tau")
            if ref["gtau"] != 0.0:
                assert _rel(got["gtau"], ref["gtau"]) < 1e-3, (variant, s, r, "gtau")
    # dataset tables: every rank holds the same replica, equal to the oracle's
    for r in range(K):
        tabs = res[r][1]
        names = ["u1", "u2"] + (["tau1", "tau2"] if "tau1" in tabs else [])
        for name in names:
            got, ref_tab = tabs[name], getattr(st, name)
            assert np.max(np.abs(got - ref_tab) / np.maximum(np.abs(ref_tab), 1e-300)) < 1e-3, (variant, r, name)


def test_nccl_fallback_matches_oracle(monkeypatch):
    # FC_PEER=0: the NCCL all-gather / all-reduce path (used when GPUs cannot map each other's
    # memory) gives the same results
    monkeypatch.setenv("FC_PEER", "0")
    B, d, N, steps = 512, 128, 8192, 2
    res, refs, st = _run(2, "fastclip_v3", B, d, N, steps)
    Bl = B // 2
    for s in range(steps):
        for r in range(2):
            got, ref = res[r][0][s], refs[s]
            assert _norm_rel(got["dE1"], ref["dE1"][r * Bl:(r + 1) * Bl]) < 2e-3
            assert _norm_rel(got["dE2"], ref["dE2"][r * Bl:(r + 1) * Bl]) < 2e-3
            assert _rel(got["loss"], ref["loss"]) < 1e-3 and _rel(got["tau"], ref["tau_new"]) < 1e-3
