"""World-size-2 gloo test of the multi-rank host logic (CPU, no GPU): each rank holds its
contiguous slice of the global batch (trainer.cpp:231-241), all-gathers the embeddings in
rank order (trainer.cpp:422-425) and the packed per-sample payload [u1|u2|t1|t2|id]
(trainer.cpp:459-487, the layout fc_table_kernel writes), and the oracle's rank-k outputs on
the gathered batch equal the single-process K=2 oracle's rows for that rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2407_01445_b200 import synthetic as S

B, D, N, K = 16, 8, 64, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=K)
    try:
        b1, b2 = S.embeddings(B, D, 5)
        ids = S.ids(B, N, 5)
        Bl = B // K
        lo = rank * Bl
        e1_loc = torch.from_numpy(S.bf16_to_f32(b1[lo:lo + Bl]).astype(np.float64))
        e2_loc = torch.from_numpy(S.bf16_to_f32(b2[lo:lo + Bl]).astype(np.float64))
        g1 = [torch.empty_like(e1_loc) for _ in range(K)]
        g2 = [torch.empty_like(e2_loc) for _ in range(K)]
        dist.all_gather(g1, e1_loc)
        dist.all_gather(g2, e2_loc)
        E1 = torch.cat(g1).numpy()
        E2 = torch.cat(g2).numpy()
        cfg = O.default_config("fastclip_v3", N)
        st = O.new_state(cfg)
        st.u1[:] = S.warm_u(N, 1)
        st.u2[:] = S.warm_u(N, 2)
        out = O.step(cfg, st, K, E1, E2, ids, 0.6, 1e-14)
        # packed payload of this rank, gathered in rank order
        pay = torch.from_numpy(np.concatenate([out["u1"][lo:lo + Bl], out["u2"][lo:lo + Bl],
                                               out["t1"][lo:lo + Bl], out["t2"][lo:lo + Bl],
                                               ids[lo:lo + Bl].astype(np.float64)]))
        gp = [torch.empty_like(pay) for _ in range(K)]
        dist.all_gather(gp, pay)
        recv = torch.stack(gp).numpy().reshape(K, 5, Bl)
        q.put((rank, out["dE1"][lo:lo + Bl], out["dE2"][lo:lo + Bl], recv, out["gtau_local"][rank]))
    finally:
        dist.destroy_process_group()


def test_two_rank_slices_match_serial_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(K)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(K)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    b1, b2 = S.embeddings(B, D, 5)
    ids = S.ids(B, N, 5)
    cfg = O.default_config("fastclip_v3", N)
    st = O.new_state(cfg)
    st.u1[:] = S.warm_u(N, 1)
    st.u2[:] = S.warm_u(N, 2)
    ref = O.step(cfg, st, K, S.bf16_to_f32(b1).astype(np.float64), S.bf16_to_f32(b2).astype(np.float64), ids,
                 0.6, 1e-14)
    Bl = B // K
    for rank, de1, de2, recv, gtl in res:
        lo = rank * Bl
        np.testing.assert_array_equal(de1, ref["dE1"][lo:lo + Bl])
        np.testing.assert_array_equal(de2, ref["dE2"][lo:lo + Bl])
        assert gtl == ref["gtau_local"][rank]
        # the gathered payload reproduces the global-batch u / tau / id vectors in order
        np.testing.assert_array_equal(recv[:, 0, :].reshape(-1), ref["u1"])
        np.testing.assert_array_equal(recv[:, 1, :].reshape(-1), ref["u2"])
        np.testing.assert_array_equal(recv[:, 4, :].reshape(-1).astype(np.int32), ids)
