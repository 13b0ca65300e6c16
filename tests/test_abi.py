"""The C ABI library loads without a GPU and exports every symbol include/fastclip_b200.h
declares; host-only entry points (defaults, schedules) match the reference."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fastclip_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|double|const char\*)\s+(fc_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    import paper_2407_01445_b200 as P
    L = P.lib()
    names = _declared()
    assert len(names) >= 40
    for n in names:
        assert hasattr(L, n), n


def test_config_defaults_match_reference_resolution():
    import paper_2407_01445_b200 as P
    v3 = P.config_defaults("fastclip_v3", 100)
    assert (v3.tau_init, v3.rho, v3.tau_lr, v3.lr_decay_enabled, v3.scale_by_tau) == (0.07, 6.5, 2e-4, 1, 1)
    v2 = P.config_defaults("fastclip_v2", 100)
    assert (v2.tau_init, v2.rho, v2.tau_lr, v2.scale_by_tau) == (0.03, 9.0, 1e-2, 1)
    v0 = P.config_defaults("fastclip_v0", 100)
    assert (v0.scale_by_tau, v0.tau_lr) == (0, 2e-4)
    v1 = P.config_defaults("fastclip_v1", 100)
    assert v1.tau_lr == 0.0
    mb = P.config_defaults("openclip_mbcl", 100)
    assert (mb.scale_by_tau, mb.rho) == (0, 0.0)
    # fabric.reduction = auto: the OpenCLIP baseline reduce-scatters, everything else gathers u
    assert mb.reduction == 1 and v3.reduction == 0 and v2.reduction == 0   # trainer.cpp:86-88
    with pytest.raises(P.FastclipError):
        P.config_defaults(9, 100)


def test_schedules_match_oracle():
    import oracle as O
    import paper_2407_01445_b200 as P
    L = O.lib("oracle")
    for t in range(0, 400, 7):
        assert P.gamma_at(t, decay_epochs=18, iters_per_epoch=11, gamma_min=0.2) == L.oc_gamma_cosine(t, 11, 18, 0.2)
    assert P.gamma_at(5, cosine=False, constant=0.6) == 0.6
    assert P.epsilon_at(3, 1e-14, 1e-8, 4) == 1e-14
    assert P.epsilon_at(4, 1e-14, 1e-8, 4) == 1e-8
    assert P.epsilon_at(40, 1e-14, 1e-8, -1) == 1e-14


def test_create_rejects_bad_shapes_without_gpu_work():
    import paper_2407_01445_b200 as P
    cfg = P.config_defaults("fastclip_v3", 100, dim=12, local_batch=16)   # dim % 8 != 0
    with pytest.raises(P.FastclipError) as e:
        P.LossStep(cfg)
    assert e.value.kind in ("Unsupported", "CudaError")


def test_temperature_step_matches_oracle():
    # opt::temperature_step (optimizers.cpp:77-83) through the C ABI (host scalar) against the
    # C restatement, over a sequence of steps incl. the projection onto tau0 and a NaN gradient
    import ctypes as C
    import oracle as O
    import paper_2407_01445_b200 as P
    L = O.lib("oracle")
    L.oc_temperature_step.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_double,
                                      C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.POINTER(C.c_double)]
    st = dict(m=0.0, v=0.0, step=0)
    m, v, s, out = C.c_double(0.0), C.c_double(0.0), C.c_int64(0), C.c_double(0.0)
    tau_a = tau_b = 0.03
    for k, g in enumerate([3.1, -2.0, 0.5, 40.0, 40.0, 40.0, -1e-3]):
        tau_a = P.temperature_step(st, tau_a, g, 2e-4 if k < 3 else 5e-2)
        assert L.oc_temperature_step(C.byref(m), C.byref(v), C.byref(s), tau_b, g, 2e-4 if k < 3 else 5e-2, 0.9, 0.999,
                                     1e-8, 0.005, C.byref(out)) == 0
        tau_b = out.value
        assert tau_a == tau_b and st["m"] == m.value and st["v"] == v.value and st["step"] == s.value
    assert tau_a == 0.005                                  # projected onto tau0
    with pytest.raises(P.FastclipError) as e:
        P.temperature_step(st, tau_a, float("nan"), 1e-3)
    assert e.value.code == 9
