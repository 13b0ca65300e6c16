"""Per-function entry point fc_g_values (engine::g_values, engine.cpp:151-176, and
engine::dtau_sums, engine.cpp:182-204) on the step's tcgen05 pass-1 kernel vs the oracle's
oc_g_values / oc_dtau_sums on the same bf16 inputs: max relative error <= 1e-3, clamp counts
equal to the oracle's (within the fp32-vs-fp64 rounding of exponents that sit on the clamp)."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from gpu_helpers import to_dev_bf16
from paper_2407_01445_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _oracle(E1, E2, t1, t2, lo, cnt):
    L = O.lib("oracle")
    DP = C.POINTER(C.c_double)
    for f in ("oc_g_values", "oc_dtau_sums"):
        getattr(L, f).argtypes = [C.c_int, C.c_int, DP, DP, DP, DP, C.c_int, C.c_int, DP, DP]
    B, d = E1.shape
    p = lambda a: a.ctypes.data_as(DP)
    g1, g2, d1, d2 = (np.zeros(cnt) for _ in range(4))
    L.oc_reset_exp_clamp_count()
    assert L.oc_g_values(B, d, p(E1), p(E2), p(t1), p(t2), lo, cnt, p(g1), p(g2)) == 0
    clamps = L.oc_exp_clamp_count()
    # dtau_sums indexes t by the GLOBAL row (engine.cpp:198-199): pass t over G with the local
    # slice's values at [lo, lo + cnt)
    T1, T2 = np.ones(B), np.ones(B)
    T1[lo:lo + cnt], T2[lo:lo + cnt] = t1, t2
    assert L.oc_dtau_sums(B, d, p(E1), p(E2), p(T1), p(T2), lo, cnt, p(d1), p(d2)) == 0
    return dict(g1=g1, g2=g2, dsum1=d1, dsum2=d2, clamps=clamps)


def _rel(a, b, floor=0.0):
    """max relative error; `floor` (a fraction of max |b|) bounds the denominator as numdiff's
    max_rel_error does (numdiff.hpp:45-56) for signed sums that can cancel."""
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), max(floor * np.max(np.abs(b)), 1e-300))))


@pytest.mark.parametrize("B,d,lo,cnt,tmin,tmax", [
    (600, 200, 128, 256, 0.02, 0.1),     # ragged B, a slice in the middle, individual temperatures
    (512, 128, 0, 512, 0.07, 0.07),      # the whole batch at one temperature (K = 1 shape)
    (384, 64, 300, 84, 0.005, 0.01),     # tau near the floor: safe_exp clamps are hit
])
def test_g_values_match_oracle(B, d, lo, cnt, tmin, tmax):
    import torch
    import paper_2407_01445_b200 as P
    b1, b2 = S.embeddings(B, d, 31)
    rng = np.random.default_rng(5)
    t1 = rng.uniform(tmin, tmax, cnt)
    t2 = rng.uniform(tmin, tmax, cnt)
    got = P.g_values(to_dev_bf16(b1), to_dev_bf16(b2), torch.from_numpy(t1).cuda(), torch.from_numpy(t2).cuda(), lo, cnt)
    ref = _oracle(S.bf16_to_f32(b1).astype(np.float64), S.bf16_to_f32(b2).astype(np.float64), t1, t2, lo, cnt)
    for k in ("g1", "g2"):   # positive sums: strict element-wise relative error
        assert _rel(got[k].cpu().numpy(), ref[k]) < 1e-3, k
    for k in ("dsum1", "dsum2"):   # signed sums of (s - S_ii) e: an anchor's sum can cancel towards 0
        assert _rel(got[k].cpu().numpy(), ref[k], floor=1e-3) < 1e-3, k
    assert got["clamps"] == pytest.approx(ref["clamps"], rel=0.02, abs=2)
    if tmin <= 0.005:
        assert ref["clamps"] > 0


def test_g_values_rejects_bad_slices():
    import torch
    import paper_2407_01445_b200 as P
    b1, b2 = S.embeddings(64, 16, 1)
    t = torch.full((32,), 0.05, dtype=torch.float64, device="cuda")
    with pytest.raises(P.FastclipError) as e:
        P.g_values(to_dev_bf16(b1), to_dev_bf16(b2), t, t, 48, 32)   # slice past the batch
    assert e.value.code == 2


def _oracle_cot(E1, E2, w1, w2, t1, t2, lo, cnt):
    L = O.lib("oracle")
    DP = C.POINTER(C.c_double)
    L.oc_embedding_cotangents.argtypes = [C.c_int, C.c_int, DP, DP, DP, DP, DP, DP, C.c_int, C.c_int, DP, DP]
    B, d = E1.shape
    p = lambda a: a.ctypes.data_as(DP)
    d1, d2 = np.zeros((cnt, d)), np.zeros((cnt, d))
    assert L.oc_embedding_cotangents(B, d, p(E1), p(E2), p(w1), p(w2), p(t1), p(t2), lo, cnt, p(d1), p(d2)) == 0
    return d1, d2


@pytest.mark.parametrize("B,d,lo,cnt,tmin,tmax", [
    (600, 200, 128, 256, 0.02, 0.1),     # ragged, middle slice, per-anchor temperatures (v2-like)
    (512, 128, 0, 512, 0.07, 0.07),      # whole batch, one temperature (v3-like)
    (384, 64, 300, 84, 0.01, 0.03),      # small tail slice
])
def test_embedding_cotangents_match_oracle(B, d, lo, cnt, tmin, tmax):
    import torch
    import paper_2407_01445_b200 as P
    b1, b2 = S.embeddings(B, d, 41)
    rng = np.random.default_rng(9)
    t1, t2 = rng.uniform(tmin, tmax, B), rng.uniform(tmin, tmax, B)
    w1, w2 = t1 / (1e-14 + 10 ** rng.uniform(-6, 0, B)), t2 / (1e-14 + 10 ** rng.uniform(-6, 0, B))
    cuda = lambda a: torch.from_numpy(a).cuda()
    de1, de2 = P.embedding_cotangents(to_dev_bf16(b1), to_dev_bf16(b2), cuda(w1), cuda(w2), cuda(t1), cuda(t2), lo, cnt)
    r1, r2 = _oracle_cot(S.bf16_to_f32(b1).astype(np.float64), S.bf16_to_f32(b2).astype(np.float64), w1, w2, t1, t2,
                         lo, cnt)
    nr = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    assert nr(de1.cpu().numpy().astype(np.float64), r1) < 2e-3
    assert nr(de2.cpu().numpy().astype(np.float64), r2) < 2e-3


def test_table_update_matches_state_semantics():
    # UTable::update + snapshot (state.cpp:45-71): fp64 EMA at the ids, snapshot in batch order,
    # untouched entries bit-identical; an id outside the table is a ShapeError (skipped)
    import torch
    import paper_2407_01445_b200 as P
    N, n = 5000, 300
    rng = np.random.default_rng(3)
    u1, u2 = S.warm_u(N, 1), S.warm_u(N, 2)
    ids = rng.choice(N, n, replace=False).astype(np.int32)
    g1, g2 = rng.uniform(0, 2, n), rng.uniform(0, 2, n)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    U1, U2 = d(u1), d(u2)
    o1, o2, status = P.table_update(U1, U2, d(ids), d(g1), d(g2), 0.6)
    r1, r2 = u1.copy(), u2.copy()
    r1[ids] = 0.4 * u1[ids] + 0.6 * g1
    r2[ids] = 0.4 * u2[ids] + 0.6 * g2
    assert status == 0
    mask = np.ones(N, bool)
    mask[ids] = False
    for got, ref in ((U1.cpu().numpy(), r1), (U2.cpu().numpy(), r2)):
        np.testing.assert_array_equal(got[mask], ref[mask])            # untouched: bit-identical
        np.testing.assert_allclose(got[ids], ref[ids], rtol=1e-14)     # fp64 EMA (FMA contraction)
    np.testing.assert_array_equal(o1.cpu().numpy(), U1.cpu().numpy()[ids])   # the snapshot is the table
    bad = ids.copy()
    bad[5] = N
    _, _, status = P.table_update(U1, U2, d(bad), d(g1), d(g2), 0.6)
    assert status == 2
    with pytest.raises(P.FastclipError):
        P.table_update(U1, U2, d(ids), d(g1), d(g2), 1.5)   # gamma outside (0, 1]


@pytest.mark.parametrize("variant", ["fastclip_v3", "fastclip_v0", "openclip_mbcl", "fastclip_v2"])
def test_grad_tau_composes_to_the_step_gradient(variant):
    # fc_g_values (dtau sums at tau^t) + fc_grad_tau on the oracle's u snapshot reproduce the
    # oracle step's G_tau (v0 / v3 / MBCL) or per-index gtau1 / gtau2 (v2), K = 1
    import torch
    import paper_2407_01445_b200 as P
    B, d, N = 384, 96, 4000
    cfg = O.default_config(variant, N)
    st = O.new_state(cfg)
    st.u1[:] = S.warm_u(N, 0)
    st.u2[:] = S.warm_u(N, 1)
    b1, b2 = S.embeddings(B, d, 12)
    ids = S.ids(B, N, 12)
    tau = st.tau
    ref = O.step(cfg, st, 1, S.bf16_to_f32(b1).astype(np.float64), S.bf16_to_f32(b2).astype(np.float64), ids, 0.6, 1e-14)
    cuda = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    gv = P.g_values(to_dev_bf16(b1), to_dev_bf16(b2), cuda(ref["t1"]), cuda(ref["t2"]), 0, B)
    out = P.grad_tau(variant, cuda(ref["u1"]), cuda(ref["u2"]), gv["dsum1"], gv["dsum2"], B, 1e-14, cfg["rho"], tau,
                     cuda(ref["t1"]), cuda(ref["t2"]), N)
    if variant == "fastclip_v2":
        # per-index terms log(eps + u) + rho + t dsum / (eps + u) can cancel to ~0 for single
        # indices, so the error is taken relative to the largest |gtau| (numdiff.hpp:45-56 floor)
        for got, r in ((out[0], ref["gtau1"]), (out[1], ref["gtau2"])):
            assert np.max(np.abs(got.cpu().numpy() - r)) <= 1e-3 * np.max(np.abs(r))
    else:
        assert abs(out - ref["gtau"]) <= 1e-3 * abs(ref["gtau"])
