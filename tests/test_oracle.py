"""The CPU restatement (oracle/fastclip_oracle.c) pinned against the reference: SPEC.md known
answers and the golden vectors produced by the reference's own translation units."""
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_2407_01445_b200 import synthetic as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_safe_exp_clamp_and_counter():
    L = O.lib("oracle")
    L.oc_reset_exp_clamp_count()
    assert L.oc_safe_exp(1.0) == math.exp(1.0)
    assert L.oc_safe_exp(61.0) == math.exp(60.0)          # losses.cpp:22-28
    assert L.oc_exp_clamp_count() == 1


def test_gamma_schedule_anchors():
    L = O.lib("oracle")
    # SPEC.md:153-ish anchors: gamma_min=0.2, E=18 -> epoch 0: 1.0, epoch 9: 0.6, >=18: 0.2
    assert L.oc_gamma_cosine(0, 10, 18, 0.2) == pytest.approx(1.0)
    assert L.oc_gamma_cosine(90, 10, 18, 0.2) == pytest.approx(0.6)
    assert L.oc_gamma_cosine(180, 10, 18, 0.2) == pytest.approx(0.2)


def test_latch_is_one_way():
    import ctypes as C
    L = O.lib("oracle")
    lat = C.c_int(0)
    assert L.oc_latch_modifier(C.byref(lat), 0.05, 0.03, 1 / 3) == 1.0
    assert L.oc_latch_modifier(C.byref(lat), 0.02, 0.03, 1 / 3) == pytest.approx(1 / 3)
    assert L.oc_latch_modifier(C.byref(lat), 0.05, 0.03, 1 / 3) == pytest.approx(1 / 3)


def test_spec_known_answers_ell_and_g():
    # ell1 with s_ij=0, s_ii=1, tau=0.5 -> e^-2; g over {1, e^-2}
    E1 = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 0.0]])
    E2 = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 0.0]])
    g1 = np.zeros(1)
    g2 = np.zeros(1)
    import ctypes as C
    L = O.lib("oracle")
    t = np.array([0.5])
    rc = L.oc_g_values(3, 2, O._ptr(E1), O._ptr(E2), O._ptr(t), O._ptr(t), 0, 1, O._ptr(g1), O._ptr(g2))
    assert rc == 0
    # anchor 0: s00=1, s01=0 -> e^-2, s02=1 -> 1 ; mean = (1+e^-2)/2 = 0.56767
    assert g1[0] == pytest.approx((1 + math.exp(-2)) / 2, rel=1e-12)
    assert g1[0] == pytest.approx(0.56767, abs=1e-5)


def test_identical_embeddings_give_zero_gradient_and_margin_tau_grad():
    # all embeddings identical -> zero w-gradient, v3 G_tau = 2log(eps+1)+2rho
    B, d, N = 8, 4, 16
    E = np.tile(np.array([[0.5, 0.5, 0.5, 0.5]]), (B, 1))
    cfg = O.default_config("fastclip_v3", N)
    st = O.new_state(cfg)
    out = O.step(cfg, st, 1, E, E, np.arange(B, dtype=np.int32), 1.0, 1e-14)
    assert np.abs(out["dE1"]).max() < 1e-15 and np.abs(out["dE2"]).max() < 1e-15
    assert out["gtau"] == pytest.approx(2 * math.log(1e-14 + 1) + 2 * 6.5, rel=1e-12)


def test_v2_symmetric_tau_grad_is_rho_over_n():
    # u = 1, nabla terms zero, rho = 9 -> 9/n
    B, d, N = 6, 4, 12
    E = np.tile(np.array([[1.0, 0.0, 0.0, 0.0]]), (B, 1))
    cfg = O.default_config("fastclip_v2", N)
    st = O.new_state(cfg)
    out = O.step(cfg, st, 1, E, E, np.arange(B, dtype=np.int32), 1.0, 1e-14)
    assert np.allclose(out["gtau1"], 9.0 / N, rtol=1e-12)


def test_update_u_known_answer():
    # gamma=0.5, u=0.4, g=0.8 -> 0.6 (g forced by identical embeddings: g=1)
    B, d, N = 4, 2, 8
    E = np.tile(np.array([[1.0, 0.0]]), (B, 1))
    cfg = O.default_config("fastclip_v1", N)
    st = O.new_state(cfg)
    st.u1[:] = 0.4
    out = O.step(cfg, st, 1, E, E, np.arange(B, dtype=np.int32), 0.5, 1e-14)
    assert np.allclose(out["u1"], 0.5 * 0.4 + 0.5 * 1.0)


def test_k_invariance_of_tau_grad():
    # all_reduce_mean of per-worker G_tau equals the serial value
    B, d, N = 16, 8, 64
    b1, b2 = S.embeddings(B, d, 3)
    E1, E2 = S.bf16_to_f32(b1).astype(np.float64), S.bf16_to_f32(b2).astype(np.float64)
    ids = S.ids(B, N, 3)
    cfg = O.default_config("fastclip_v0", N)
    outs = []
    for K in (1, 2, 4):
        st = O.new_state(cfg)
        st.u1[:] = S.warm_u(N, 1)
        st.u2[:] = S.warm_u(N, 2)
        outs.append(O.step(cfg, st, K, E1, E2, ids, 0.6, 1e-14))
    for o in outs[1:]:
        assert o["gtau"] == pytest.approx(outs[0]["gtau"], rel=1e-12)
        # rank-k cotangents carry the K x scale (trainer.cpp:540-546 divides by K later)


def _replay(path, backend="oracle"):
    z = np.load(path)
    cfg = {k[4:]: z[k].item() for k in z.files if k.startswith("cfg_")}
    cfg["variant"] = int(cfg["variant"])
    cfg["n_train"] = int(cfg["n_train"])
    for k in ("lr_decay_enabled", "scale_by_tau"):
        cfg[k] = int(cfg[k])
    st = O.new_state(cfg)
    st.u1[:] = z["state0_u1"]
    st.u2[:] = z["state0_u2"]
    K = int(z["K"])
    res = []
    for s in range(int(z["steps"])):
        E1 = S.bf16_to_f32(z[f"s{s}_E1bits"]).astype(np.float64)
        E2 = S.bf16_to_f32(z[f"s{s}_E2bits"]).astype(np.float64)
        out = O.step(cfg, st, K, E1, E2, z[f"s{s}_ids"], float(z["gamma"]), float(z["eps"]), backend)
        res.append((s, out, st.copy()))
    return z, res


def test_oracle_matches_reference_golden(golden_files):
    assert len(golden_files) >= 10
    for path in golden_files:
        z, res = _replay(path)
        for s, out, st in res:
            for k in ("dE1", "dE2", "g1", "g2", "u1", "u2", "t1", "t2", "gtau1", "gtau2", "gtau_local"):
                ref = z[f"s{s}_{k}"]
                np.testing.assert_allclose(out[k], ref, rtol=1e-12, atol=1e-300, err_msg=f"{path} s{s} {k}")
            for k in ("gtau", "tau_new", "loss"):
                assert out[k] == pytest.approx(float(z[f"s{s}_{k}"]), rel=1e-12), (path, s, k)
            assert out["clamps_g"] == int(z[f"s{s}_clamps_g"])
            if st.individual:
                np.testing.assert_allclose(st.tau1, z[f"s{s}_tau1_after"], rtol=1e-12)
                np.testing.assert_allclose(st.tau2, z[f"s{s}_tau2_after"], rtol=1e-12)
        np.testing.assert_array_equal(res[-1][2].u1, z["state_end_u1"])


def test_golden_clamp_case_exercises_safe_exp(golden_files):
    z = np.load([p for p in golden_files if p.endswith("_s11.npz")][0])
    assert int(z["s0_clamps_g"]) > 0


@pytest.mark.skipif(not os.path.exists(O.REF_SO), reason="reference build (oracle/_ref) absent")
def test_oracle_matches_reference_live():
    B, d, N = 24, 8, 50
    for var in O.VARIANTS:
        b1, b2 = S.embeddings(B, d, 42)
        E1, E2 = S.bf16_to_f32(b1).astype(np.float64), S.bf16_to_f32(b2).astype(np.float64)
        ids = S.ids(B, N, 42)
        cfg = O.default_config(var, N)
        a_st, b_st = O.new_state(cfg), O.new_state(cfg)
        for K in (1, 3):
            a = O.step(cfg, a_st, K, E1, E2, ids, 0.7, 1e-14, "oracle")
            b = O.step(cfg, b_st, K, E1, E2, ids, 0.7, 1e-14, "ref")
            for k in ("dE1", "dE2", "g1", "g2", "u1", "u2"):
                np.testing.assert_allclose(a[k], b[k], rtol=1e-12, err_msg=f"{var} K{K} {k}")
            assert a["tau_new"] == b["tau_new"]


@pytest.mark.parametrize("variant", ["fastclip_v3", "fastclip_v2", "fastclip_v1", "fastclip_v0", "openclip_mbcl",
                                     "sogclr", "isogclr"])
@pytest.mark.parametrize("K", [1, 2, 4])
def test_vectorised_oracle_matches_c_oracle(variant, K):
    # oracle/oracle_np.py (the full-size checker of tests/test_gpu_fullsize.py) against the C
    # restatement: 3 chained steps from warm tables, every output and the updated state
    import oracle_np as ON
    B, d, N = 96, 24, 500
    for tau_init in (None, 0.005):       # 0.005: the tau floor, safe_exp clamps are hit
        over = {} if tau_init is None else dict(tau_init=tau_init)
        cfg = O.default_config(variant, N, **over)
        a, b = O.new_state(cfg), O.new_state(cfg)
        a.u1[:] = b.u1[:] = S.warm_u(N, 0)
        a.u2[:] = b.u2[:] = S.warm_u(N, 1)
        for s in range(3):
            b1, b2 = S.embeddings(B, d, 5 + s)
            ids = S.ids(B, N, 5 + s)
            E1 = S.bf16_to_f32(b1).astype(np.float64)
            E2 = S.bf16_to_f32(b2).astype(np.float64)
            r1 = O.step(cfg, a, K, E1, E2, ids, 0.6, 1e-14)
            r2 = ON.step(cfg, b, K, E1, E2, ids, 0.6, 1e-14)
            for k in ("dE1", "dE2", "g1", "g2", "u1", "u2", "gtau1", "gtau2", "gtau_local"):
                x, y = np.asarray(r1[k]), np.asarray(r2[k])
                assert np.max(np.abs(x - y)) <= 1e-12 * max(np.max(np.abs(x)), 1e-300), (variant, K, s, k)
            for k in ("loss", "gtau", "tau_new"):
                assert abs(r1[k] - r2[k]) <= 1e-12 * abs(r1[k]) + 1e-300, (variant, K, s, k)
            assert r1["clamps_g"] == r2["clamps_g"]
        for t in ("u1", "u2", "tau1", "tau2", "m1", "v1", "m2", "v2"):
            x = getattr(a, t)
            if x is not None:
                assert np.max(np.abs(x - getattr(b, t))) <= 1e-12 * max(np.max(np.abs(x)), 1e-300), (variant, K, t)
        if a.s1 is not None:
            np.testing.assert_array_equal(a.s1, b.s1)
            np.testing.assert_array_equal(a.s2, b.s2)
        assert (a.tau, a.tau_step, a.latched) == pytest.approx((b.tau, b.tau_step, b.latched), rel=1e-12)
