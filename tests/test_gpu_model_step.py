"""The model-side step after the loss step on the B200 against the
reference: the tower forward / vjp through the normalisation Jacobian (encoder.cpp:98-177, via the
finite-difference-pinned restatement oracle_np.tower_*), the reference's own opt::adamw_step /
lamb_step (optimizers.cpp:33-63, oracle/_ref), and the composed step x -> e -> loss step -> dE ->
vjp -> AdamW."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import oracle_np as ON
from gpu_helpers import gpu_cfg
from paper_2407_01445_b200 import synthetic as S

pytestmark = pytest.mark.gpu
DP = C.POINTER(C.c_double)
LP = C.POINTER(C.c_longlong)


def _t(a, dtype=None):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda() if dtype is None else \
        torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


@pytest.mark.parametrize("kind,d_hidden", [(0, 0), (1, 48)])
def test_tower_forward_and_vjp_match_reference(kind, d_hidden):
    import paper_2407_01445_b200 as P
    rng = np.random.default_rng(4 + kind)
    rows, d_in, d_out = 300, 40, 64
    n = P.fastclip.tower_param_count(kind, d_in, d_hidden, d_out)
    theta = rng.standard_normal(n) * 0.3
    x = rng.standard_normal((rows, d_in))
    tape = P.fastclip.tower_forward(kind, _t(theta), _t(x), d_hidden, d_out)
    ref = ON.tower_forward(kind, theta, x, d_hidden, d_out)
    np.testing.assert_allclose(tape["e"].cpu().numpy(), ref["e"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(tape["znorm"].cpu().numpy(), ref["znorm"], rtol=1e-13)
    cot = rng.standard_normal((rows, d_out)).astype(np.float32)
    g = _t(np.zeros(n))
    P.fastclip.tower_vjp(kind, _t(theta), tape, _t(cot), g)
    gr = ON.tower_vjp(kind, theta, ref, cot.astype(np.float64))
    got = g.cpu().numpy()
    assert np.max(np.abs(got - gr)) <= 1e-12 * np.max(np.abs(gr))


def test_adamw_is_bit_exact_with_reference():
    import paper_2407_01445_b200 as P
    L = O.lib("ref")
    rng = np.random.default_rng(1)
    n = 10_000
    theta, m, v = rng.standard_normal(n), rng.standard_normal(n) * 0.1, rng.random(n) * 0.01
    state = {"step": 7}
    dt, dm, dv = _t(theta), _t(m), _t(v)
    for k in range(3):
        g = rng.standard_normal(n)
        assert P.fastclip.adamw_step(dt, dm, dv, state, _t(g), 1e-3, weight_decay=0.1) == 0
        stp = C.c_longlong(7 + k)
        assert L.ref_adamw_step(n, theta.ctypes.data_as(DP), m.ctypes.data_as(DP), v.ctypes.data_as(DP),
                                C.byref(stp), g.ctypes.data_as(DP), 1e-3, 0.9, 0.999, 1e-8, 0.1) == 0
        assert state["step"] == stp.value
    np.testing.assert_array_equal(dt.cpu().numpy(), theta)
    np.testing.assert_array_equal(dm.cpu().numpy(), m)
    np.testing.assert_array_equal(dv.cpu().numpy(), v)
    # NumericError on a non-finite gradient (optimizers.cpp:13): nothing changes
    bad = rng.standard_normal(n)
    bad[17] = np.nan
    before = dt.cpu().numpy().copy()
    assert P.fastclip.adamw_step(dt, dm, dv, state, _t(bad), 1e-3) == 9
    np.testing.assert_array_equal(dt.cpu().numpy(), before)


@pytest.mark.parametrize("force", [False, True])
def test_lamb_matches_reference(force):
    import paper_2407_01445_b200 as P
    L = O.lib("ref")
    rng = np.random.default_rng(2)
    segs = [(0, 2560), (2560, 40), (2600, 5000), (7600, 1)]
    n = 7601
    theta, m, v = rng.standard_normal(n), np.zeros(n), np.zeros(n)
    theta[2560:2600] = 0.0   # a zero layer: |th| = 0 -> ratio 0 unless forced
    state = {"step": 0}
    dt, dm, dv = _t(theta), _t(m), _t(v)
    off = np.array([o for o, _ in segs], np.int64)
    ln = np.array([s for _, s in segs], np.int64)
    for k in range(3):
        g = rng.standard_normal(n)
        assert P.fastclip.lamb_step(dt, dm, dv, state, _t(g), 1e-2, segs, weight_decay=0.01, force_alpha_one=force) == 0
        stp = C.c_longlong(k)
        assert L.ref_lamb_step(n, theta.ctypes.data_as(DP), m.ctypes.data_as(DP), v.ctypes.data_as(DP), C.byref(stp),
                               g.ctypes.data_as(DP), 1e-2, 0.9, 0.999, 1e-8, 0.01, len(segs), off.ctypes.data_as(LP),
                               ln.ctypes.data_as(LP), int(force)) == 0
    np.testing.assert_array_equal(dm.cpu().numpy(), m)   # moments: elementwise, bit-exact
    np.testing.assert_array_equal(dv.cpu().numpy(), v)
    got = dt.cpu().numpy()   # per-layer norms are tree sums here, sequential in the reference
    assert np.max(np.abs(got - theta) / np.maximum(np.abs(theta), 1e-12)) < 1e-12


def test_composed_model_step_matches_reference():
    # x -> tower forward -> bf16 e -> loss step -> dE -> tower vjp -> AdamW, against the same chain
    # on the reference side (oracle step on the bf16 embeddings, restated vjp, reference AdamW)
    import paper_2407_01445_b200 as P
    L = O.lib("ref")
    rng = np.random.default_rng(7)
    B, d_in, d, N = 256, 32, 64, 4096
    n1 = P.fastclip.tower_param_count(0, d_in, 0, d)
    theta = rng.standard_normal(2 * n1) * 0.2
    xi, xt = rng.standard_normal((B, d_in)), rng.standard_normal((B, d_in))
    dth = _t(theta)
    ti = P.fastclip.tower_forward(0, dth[:n1], _t(xi), 0, d)
    tt = P.fastclip.tower_forward(0, dth[n1:], _t(xt), 0, d)
    ocfg = O.default_config("fastclip_v3", N)
    step = P.LossStep(gpu_cfg(ocfg, d, B))
    ids = S.ids(B, N, 3)
    import torch
    de1, de2 = step.step(ti["e_bf16"], tt["e_bf16"], torch.from_numpy(ids).cuda(), 0.6, 1e-14)
    grad = _t(np.zeros(2 * n1))
    P.fastclip.tower_vjp(0, dth[:n1], ti, de1, grad[:n1])
    P.fastclip.tower_vjp(0, dth[n1:], tt, de2, grad[n1:])
    step.grad_allreduce_mean(grad)   # world 1: identity
    dm, dv = _t(np.zeros(2 * n1)), _t(np.zeros(2 * n1))
    assert P.fastclip.adamw_step(dth, dm, dv, {"step": 0}, grad, 1e-3) == 0
    # reference chain
    ri = ON.tower_forward(0, theta[:n1], xi, 0, d)
    rt = ON.tower_forward(0, theta[n1:], xt, 0, d)
    E1 = S.bf16_to_f32(S.bf16_round(ri["e"].astype(np.float32))).astype(np.float64)
    E2 = S.bf16_to_f32(S.bf16_round(rt["e"].astype(np.float32))).astype(np.float64)
    np.testing.assert_array_equal(ti["e_bf16"].view(torch.int16).cpu().numpy().view(np.uint16),
                                  S.bf16_round(ri["e"].astype(np.float32)))
    st = O.new_state(ocfg)
    ref = O.step(ocfg, st, 1, E1, E2, ids, 0.6, 1e-14)
    g_ref = np.concatenate([ON.tower_vjp(0, theta[:n1], ri, ref["dE1"]), ON.tower_vjp(0, theta[n1:], rt, ref["dE2"])])
    gg = grad.cpu().numpy()
    assert np.linalg.norm(gg - g_ref) <= 1e-3 * np.linalg.norm(g_ref)   # the dE tolerance carries through
    th_ref, m_ref, v_ref = theta.copy(), np.zeros(2 * n1), np.zeros(2 * n1)
    stp = C.c_longlong(0)
    assert L.ref_adamw_step(2 * n1, th_ref.ctypes.data_as(DP), m_ref.ctypes.data_as(DP), v_ref.ctypes.data_as(DP),
                            C.byref(stp), g_ref.ctypes.data_as(DP), 1e-3, 0.9, 0.999, 1e-8, 0.0) == 0
    upd, upd_ref = dth.cpu().numpy() - theta, th_ref - theta
    assert np.linalg.norm(upd - upd_ref) <= 1e-2 * np.linalg.norm(upd_ref)
