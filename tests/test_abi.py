"""The C ABI library loads without a GPU and exports every symbol include/fastclip_b200.h
declares; host-only entry points (defaults, schedules) match the reference."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fastclip_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|double|const char\*)\s+(fc_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    import paper_2407_01445_b200 as P
    L = P.lib()
    names = _declared()
    assert len(names) >= 18
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
