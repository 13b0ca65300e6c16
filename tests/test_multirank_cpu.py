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


def _plan_rs_worker(rank, port, q):
    import ctypes as C
    import paper_2407_01445_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=K)
    try:
        # (1) the product's BatchPlan: each rank's contiguous slice (trainer.cpp:231-241), gathered
        # in rank order, is the global batch
        plan = P.BatchPlan(64, B, 9)
        loc = torch.from_numpy(plan.local_batch(3, 1, rank, K).astype(np.int64))
        parts = [torch.empty_like(loc) for _ in range(K)]
        dist.all_gather(parts, loc)
        glob = torch.cat(parts).numpy()
        # (2) openclip_rs through a real reduce-scatter: this rank's rs partials from the
        # reference's engine::rs_partial_cotangents (engine.cpp:123-144), reduce_scatter_mean over
        # the ranks, scaled by rs_shard_scale (engine.cpp:146-149) and added to the anchor part
        L = O.lib("ref")
        b1, b2 = S.embeddings(B, D, 6)
        E1 = S.bf16_to_f32(b1).astype(np.float64)
        E2 = S.bf16_to_f32(b2).astype(np.float64)
        rng = np.random.default_rng(2)
        w1, w2 = rng.uniform(0.5, 2.0, B), rng.uniform(0.5, 2.0, B)
        t1 = t2 = np.full(B, 0.07)
        Bl = B // K
        lo = rank * Bl
        mask = np.zeros(B)
        mask[lo:lo + Bl] = 1.0
        DP = C.POINTER(C.c_double)
        p = lambda a: a.ctypes.data_as(DP)
        fe1, fe2 = np.zeros((B, D)), np.zeros((B, D))
        lw1, lw2 = w1 * mask, w2 * mask   # trainer.cpp:513-518: local weights only
        assert L.ref_rs_partials(B, D, p(E1), p(E2), p(lw1), p(lw2), p(t1), p(t2), lo, Bl, p(fe1), p(fe2)) == 0
        out = []
        for f in (fe1, fe2):
            shard = torch.empty(Bl * D, dtype=torch.float64)
            dist.reduce_scatter(shard, [torch.from_numpy(f[k * Bl:(k + 1) * Bl].ravel().copy()) for k in range(K)])
            out.append(shard.numpy().reshape(Bl, D) / K * L.ref_rs_shard_scale(K, Bl, B))
        q.put((rank, glob, out[0], out[1]))
    finally:
        dist.destroy_process_group()


def test_two_rank_batch_plan_and_reduce_scatter_strategy():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_rs_worker, args=(r, port, q)) for r in range(K)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(K)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import ctypes as C
    import paper_2407_01445_b200 as P
    L = O.lib("ref")
    ref_glob = np.empty(B, np.int32)
    assert L.ref_batch_plan_local(64, B, 9, 3, 1, 0, 1, ref_glob.ctypes.data_as(C.POINTER(C.c_int))) == 0
    b1, b2 = S.embeddings(B, D, 6)
    E1 = S.bf16_to_f32(b1).astype(np.float64)
    E2 = S.bf16_to_f32(b2).astype(np.float64)
    rng = np.random.default_rng(2)
    w1, w2 = rng.uniform(0.5, 2.0, B), rng.uniform(0.5, 2.0, B)
    t = np.full(B, 0.07)
    DP = C.POINTER(C.c_double)
    p = lambda a: a.ctypes.data_as(DP)
    Bl = B // K
    for rank, glob, rs1, rs2 in res:
        np.testing.assert_array_equal(glob, ref_glob)
        # reduction-strategy equivalence: anchor part + reduce-scattered contrast
        # part = the fastclip strategy's full cotangents of engine::embedding_cotangents
        full1, full2 = np.zeros((Bl, D)), np.zeros((Bl, D))
        assert L.ref_embedding_cotangents(B, D, p(E1), p(E2), p(w1), p(w2), p(t), p(t), rank * Bl, Bl, p(full1),
                                          p(full2)) == 0
        # the reference's anchor part = full minus the contrast part; the contrast part of this
        # rank's rows is exactly what the reduce-scatter delivers
        anc1, anc2 = np.zeros((Bl, D)), np.zeros((Bl, D))
        wz = np.zeros(B)
        mask = np.zeros(B)
        mask[rank * Bl:(rank + 1) * Bl] = 1.0
        assert L.ref_embedding_cotangents(B, D, p(E1), p(E2), p(w1 * mask), p(w2 * mask), p(t), p(t), rank * Bl, Bl,
                                          p(anc1), p(anc2)) == 0
        # w masked to the local rows: embedding_cotangents = anchor part + the LOCAL anchors'
        # contrast terms; the remote anchors' contrast terms come from the other rank's partials
        got1 = anc1 + rs1 - _local_contrast(L, E1, E2, w1 * mask, w2 * mask, t, rank * Bl, Bl, 0)
        got2 = anc2 + rs2 - _local_contrast(L, E1, E2, w1 * mask, w2 * mask, t, rank * Bl, Bl, 1)
        np.testing.assert_allclose(got1, full1, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(got2, full2, rtol=1e-12, atol=1e-15)
        del wz


def _local_contrast(L, E1, E2, w1, w2, t, lo, cnt, which):
    """This rank's OWN anchors' contributions to its own rows as reduce-scattered (the rows of
    its partials that the reduce-scatter returns to itself), scaled like the shard."""
    import ctypes as C
    DP = C.POINTER(C.c_double)
    p = lambda a: a.ctypes.data_as(DP)
    B_, D_ = E1.shape
    fe1, fe2 = np.zeros((B_, D_)), np.zeros((B_, D_))
    assert L.ref_rs_partials(B_, D_, p(E1), p(E2), p(w1), p(w2), p(t), p(t), lo, cnt, p(fe1), p(fe2)) == 0
    f = fe1 if which == 0 else fe2
    return f[lo:lo + cnt] / K * L.ref_rs_shard_scale(K, cnt, B_)
