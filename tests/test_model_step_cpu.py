"""CPU pins of the model-side restatement (oracle_np.tower_forward / tower_vjp, encoder.cpp:98-177):
central finite differences of L(theta) = sum(cot o e(theta)) equal the restated vjp, as the
reference's own grad-check suite asks (SPEC finite-difference oracle, numdiff.hpp:13-56)."""
import numpy as np
import pytest

import oracle_np as ON


@pytest.mark.parametrize("kind,d_hidden", [(0, 0), (1, 7)])
def test_restated_vjp_is_the_gradient(kind, d_hidden):
    rng = np.random.default_rng(kind)
    rows, d_in, d_out = 5, 6, 4
    n = d_out * d_in + d_out if kind == 0 else d_hidden * d_in + d_hidden + d_out * d_hidden + d_out
    theta = rng.standard_normal(n) * 0.5
    x = rng.standard_normal((rows, d_in))
    cot = rng.standard_normal((rows, d_out))
    g = ON.tower_vjp(kind, theta, ON.tower_forward(kind, theta, x, d_hidden, d_out), cot)
    h = 1e-6   # numdiff.hpp's central-difference step
    fd = np.empty(n)
    for i in range(n):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += h
        tm[i] -= h
        fp = np.sum(cot * ON.tower_forward(kind, tp, x, d_hidden, d_out)["e"])
        fm = np.sum(cot * ON.tower_forward(kind, tm, x, d_hidden, d_out)["e"])
        fd[i] = (fp - fm) / (2 * h)
    assert np.max(np.abs(fd - g) / np.maximum(np.abs(g), 1e-3)) < 1e-4   # SPEC.md:701 (rel 1e-4)
