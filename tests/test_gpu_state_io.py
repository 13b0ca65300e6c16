"""On-disk state in the reference's formats, checked against the
reference's own readers / writers (state.cpp:73-162, checkpoint.cpp:57-114 in oracle/_ref):
the device u / tau / Adam tables round-trip bit-exactly, FCK1 files are byte-identical after a
reference read + write, and a resumed run continues bit-identically."""
import ctypes as C
import filecmp

import numpy as np
import pytest

import oracle as O
from gpu_helpers import gpu_cfg, to_dev_bf16
from paper_2407_01445_b200 import synthetic as S

pytestmark = pytest.mark.gpu
DP = C.POINTER(C.c_double)
LP = C.POINTER(C.c_longlong)


def _ref():
    try:
        return O.lib("ref")
    except FileNotFoundError:
        pytest.skip("reference build (oracle/_ref) absent")


def _stepper(variant, N=3000, B=128, d=64, seed=0):
    import paper_2407_01445_b200 as P
    ocfg = O.default_config(variant, N)
    st = P.LossStep(gpu_cfg(ocfg, d, B))
    st.load_tables(u1=S.warm_u(N, seed), u2=S.warm_u(N, seed + 1))
    return st


def _run(st, steps, seed0, N=3000, B=128, d=64):
    import torch
    outs = []
    for s in range(steps):
        b1, b2 = S.embeddings(B, d, seed0 + s)
        ids = torch.from_numpy(S.ids(B, N, seed0 + s)).cuda()
        de1, de2 = st.step(to_dev_bf16(b1), to_dev_bf16(b2), ids, 0.6, 1e-14)
        outs.append((de1.cpu().numpy().copy(), de2.cpu().numpy().copy(), st.scalars()))
    return outs


def _p(a, t=DP):
    return a.ctypes.data_as(t)


@pytest.mark.parametrize("variant", ["fastclip_v3", "fastclip_v2"])
def test_table_stream_matches_reference(variant, tmp_path):
    L = _ref()
    N = 3000
    st = _stepper(variant, N)
    _run(st, 2, 10)
    path = str(tmp_path / "tables.bin")
    st.write_tables(path)
    tabs = st.tables()
    indiv = "tau1" in tabs
    ref = {k: np.zeros(N) for k in ("u1", "u2", "tau1", "tau2", "m1", "v1", "m2", "v2")}
    ref.update(s1=np.zeros(N, np.int64), s2=np.zeros(N, np.int64))
    tau0 = C.c_double()
    assert L.ref_tables_read(path.encode(), N, int(indiv), _p(ref["u1"]), _p(ref["u2"]), _p(ref["tau1"]),
                             _p(ref["tau2"]), C.byref(tau0), _p(ref["m1"]), _p(ref["v1"]), _p(ref["s1"], LP),
                             _p(ref["m2"]), _p(ref["v2"]), _p(ref["s2"], LP)) == 0
    for k in tabs:   # the reference reads exactly the device tables
        np.testing.assert_array_equal(tabs[k], ref[k], err_msg=k)
    # a stream written by the reference's writers loads bit-exactly
    rng = np.random.default_rng(3)
    new = {k: rng.random(N) for k in ("u1", "u2", "tau1", "tau2", "m1", "v1", "m2", "v2")}
    new.update(s1=rng.integers(0, 50, N).astype(np.int64), s2=rng.integers(0, 50, N).astype(np.int64))
    path2 = str(tmp_path / "tables_ref.bin")
    assert L.ref_tables_write(path2.encode(), N, _p(new["u1"]), _p(new["u2"]), _p(new["tau1"]) if indiv else None,
                              _p(new["tau2"]), st.cfg.tau0, _p(new["m1"]), _p(new["v1"]), _p(new["s1"], LP),
                              _p(new["m2"]), _p(new["v2"]), _p(new["s2"], LP)) == 0
    st.read_tables(path2)
    got = st.tables()
    for k in got:
        np.testing.assert_array_equal(got[k], new[k], err_msg=k)
    # and our writer reproduces the reference's file byte for byte
    path3 = str(tmp_path / "tables_again.bin")
    st.write_tables(path3)
    assert filecmp.cmp(path2, path3, shallow=False)


@pytest.mark.parametrize("variant", ["fastclip_v3", "fastclip_v2"])
def test_checkpoint_matches_reference(variant, tmp_path):
    L = _ref()
    N = 3000
    st = _stepper(variant, N)
    _run(st, 3, 20)
    rng = np.random.default_rng(1)
    n_params = 2 * (16 * 8 + 16)
    model = dict(seed=77, next_epoch=3, global_step=1234, image_shape=(0, 8, 0, 16), text_shape=(0, 8, 0, 16),
                 params=rng.standard_normal(n_params), opt_m=rng.standard_normal(n_params),
                 opt_v=rng.random(n_params), opt_step=1234)
    path = str(tmp_path / "ck.fck1")
    st.write_checkpoint(path, model)
    path2 = str(tmp_path / "ck_ref.fck1")
    assert L.ref_checkpoint_rewrite(path.encode(), path2.encode()) == 0
    assert filecmp.cmp(path, path2, shallow=False)   # the reference reads and re-writes it unchanged
    seed, ep, gs, npar, ts_step = C.c_ulonglong(), C.c_longlong(), C.c_longlong(), C.c_longlong(), C.c_longlong()
    tau, tm, tv = C.c_double(), C.c_double(), C.c_double()
    lat, hi = C.c_int(), C.c_int()
    assert L.ref_checkpoint_fields(path.encode(), C.byref(seed), C.byref(ep), C.byref(gs), C.byref(npar), C.byref(tau),
                                   C.byref(tm), C.byref(tv), C.byref(ts_step), C.byref(lat), C.byref(hi)) == 0
    ts = st.tau_state()
    assert (seed.value, ep.value, gs.value, npar.value) == (77, 3, 1234, n_params)
    assert (tau.value, tm.value, tv.value, ts_step.value, lat.value) == (ts["tau"], ts["m"], ts["v"], ts["step"],
                                                                          ts["latched"])
    assert hi.value == int(variant == "fastclip_v2")
    # a checkpoint written by the reference restores into a fresh context
    if variant == "fastclip_v3":
        u1, u2 = rng.random(N), rng.random(N)
        p3 = str(tmp_path / "made.fck1")
        pm = rng.standard_normal(n_params)
        assert L.ref_checkpoint_make(p3.encode(), 5, 6, 7, 8, 16, n_params, _p(pm), _p(pm), _p(pm), 9, 0.0421, 0.5,
                                     0.25, 11, 1, N, _p(u1), _p(u2)) == 0
        st2 = _stepper(variant, N, seed=9)
        m = st2.read_checkpoint(p3)
        assert (m["seed"], m["next_epoch"], m["global_step"], m["opt_step"]) == (5, 6, 7, 9)
        np.testing.assert_array_equal(m["params"], pm)
        t2 = st2.tables()
        np.testing.assert_array_equal(t2["u1"], u1)
        np.testing.assert_array_equal(t2["u2"], u2)
        ts2 = st2.tau_state()
        assert (ts2["tau"], ts2["m"], ts2["v"], ts2["step"], ts2["latched"]) == (0.0421, 0.5, 0.25, 11, 1)


@pytest.mark.parametrize("variant", ["fastclip_v3", "fastclip_v2"])
def test_resume_continues_bit_identically(variant, tmp_path):
    # trainer.cpp:340-362: a run split at a checkpoint continues exactly like the unsplit run
    # (tables and temperature state bit-identical; dE to the GEMM's float reassociation)
    a = _stepper(variant)
    full = _run(a, 4, 30)
    b = _stepper(variant)
    _run(b, 2, 30)
    path = str(tmp_path / "mid.fck1")
    b.write_checkpoint(path)
    c = _stepper(variant, seed=5)   # different initial tables: everything must come from the file
    c.read_checkpoint(path)
    tail = _run(c, 2, 32)
    ta, tc = a.tables(), c.tables()
    for k in ta:
        np.testing.assert_array_equal(ta[k], tc[k], err_msg=k)
    assert a.tau_state() == c.tau_state()
    for (d1, d2, sa), (e1, e2, sc) in zip(full[2:], tail):
        assert np.linalg.norm(d1 - e1) <= 1e-6 * np.linalg.norm(d1)
        assert np.linalg.norm(d2 - e2) <= 1e-6 * np.linalg.norm(d2)
        assert sa.loss == sc.loss and sa.tau == sc.tau
