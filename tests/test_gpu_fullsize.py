"""GPU parity at the BASELINE.json shapes (full size, one GPU): the B200 step through the C ABI
against the vectorised fp64 restatement oracle/oracle_np.py (pinned to the C oracle, and through
it to the reference's own translation units, by tests/test_oracle.py). Same tolerances as
tests/test_gpu_step.py: g, u, loss, tau, G_tau max rel 1e-3; dE norm-relative 1e-3; table
indexing bit-exact (untouched entries identical, touched entries at the right ids).

Shapes: the north star (v3, B = 5120, d = 512, N = 2.7M); config 2's global batch on one GPU
(v2, B = 8192, N = 9.1M); config 3 (v3, d = 768, N = 2.7M and the full N = 315M); config 4 (v0 and v2, B = 4096,
d = 1024); config 5's next size up (v3, B = 16384)."""
import numpy as np
import pytest

import oracle_np as ON
from gpu_helpers import norm_rel, rel, run_pair
from paper_2407_01445_b200 import synthetic as S

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _check_full(res, tabs, st, what, ids_of):
    for i, (got, ref) in enumerate(res):
        w = f"{what} step {i}"
        for k in ("g1", "g2", "u1", "u2"):
            assert rel(got[k], ref[k]) < TOL, (w, k, rel(got[k], ref[k]))
        assert abs(got["loss"] - ref["loss"]) <= TOL * abs(ref["loss"]), (w, got["loss"], ref["loss"])
        assert abs(got["tau_new"] - ref["tau_new"]) <= TOL * abs(ref["tau_new"]), (w, got["tau_new"], ref["tau_new"])
        if ref["gtau"] != 0.0:
            assert abs(got["gtau"] - ref["gtau"]) <= TOL * abs(ref["gtau"]), (w, got["gtau"], ref["gtau"])
        assert norm_rel(got["dE1"], ref["dE1"]) < TOL, (w, norm_rel(got["dE1"], ref["dE1"]))
        assert norm_rel(got["dE2"], ref["dE2"]) < TOL, (w, norm_rel(got["dE2"], ref["dE2"]))
    # dataset tables after all steps: untouched entries bit-identical, touched ids within 1e-3
    touched = np.zeros(len(st.u1), bool)
    for i in range(len(res)):
        touched[ids_of(i)] = True
    for name in ("u1", "u2") + (("tau1", "tau2") if "tau1" in tabs else ()):
        got, ref = tabs[name], getattr(st, name)
        np.testing.assert_array_equal(got[~touched], ref[~touched])
        assert rel(got[touched], ref[touched]) < TOL, (what, name)

@pytest.mark.parametrize("variant,B,d,N,steps", [
    ("fastclip_v3", 5120, 512, 2_700_000, 2),    # north star / BASELINE configs[1]
    ("fastclip_v2", 8192, 512, 9_100_000, 1),    # config 2's global batch at K = 1
    ("fastclip_v3", 5120, 768, 2_700_000, 1),    # config 3's width
    ("fastclip_v3", 5120, 768, 315_000_000, 1),  # config 3 in full: LAION-scale u tables (2 x 2.5 GB fp64)
    ("fastclip_v0", 4096, 1024, 2_700_000, 1),   # config 4
    ("fastclip_v2", 4096, 1024, 2_700_000, 1),   # config 4
    ("fastclip_v3", 16384, 512, 2_700_000, 1),   # config 5 (B = 16k)
])
def test_full_size_matches_oracle(variant, B, d, N, steps):
    res, tabs, st, step = run_pair(variant, B=B, d=d, N=N, steps=steps, seed=29, checker=ON.step)
    step.close()
    _check_full(res, tabs, st, f"{variant} B={B} d={d}", lambda s: S.ids(B, N, 29 * 1000 + s))
