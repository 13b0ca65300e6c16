"""Generates tests/golden/*.npz from the REFERENCE's own code (oracle/_ref, the reference's
hot-path translation units compiled against the Eigen-subset shim). Run in the dev container
(needs /root/reference for `make -C oracle ref`):

    make -C oracle && python tests/golden/make_golden.py

Each fixture holds the synthetic inputs (bf16 bit patterns), the table state before the
steps, and per step the reference outputs; the oracle restatement and the GPU path are both
checked against these.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
from paper_2407_01445_b200 import synthetic as S  # noqa: E402

CASES = [
    # (variant, K, B, d, N, steps, gamma, eps, seed)
    ("fastclip_v3", 1, 32, 16, 128, 3, 0.6, 1e-14, 1),
    ("fastclip_v3", 2, 32, 16, 128, 3, 0.6, 1e-14, 2),
    ("fastclip_v0", 1, 24, 16, 96, 2, 1.0, 1e-14, 3),
    ("fastclip_v1", 2, 24, 8, 96, 2, 0.2, 1e-14, 4),
    ("fastclip_v2", 1, 32, 16, 64, 3, 0.6, 1e-14, 5),
    ("fastclip_v2", 4, 32, 16, 64, 2, 0.6, 1e-14, 6),
    ("sogclr", 1, 20, 8, 40, 2, 0.9, 1e-14, 7),
    ("isogclr", 2, 20, 8, 40, 2, 0.9, 1e-14, 8),
    ("openclip_mbcl", 1, 24, 16, 48, 2, 1.0, 1e-14, 9),
    ("openclip_mbcl", 2, 24, 16, 48, 2, 1.0, 1e-14, 10),
    # tau at the floor: exponent clamps (safe_exp, losses.cpp:22-28) are exercised
    ("fastclip_v3", 1, 32, 16, 128, 2, 0.6, 1e-14, 11, dict(tau_init=0.005)),
]


def make(case):
    var, K, B, d, N, steps, gamma, eps, seed = case[:9]
    over = case[9] if len(case) > 9 else {}
    cfg = O.default_config(var, N, **over)
    st = O.new_state(cfg)
    st.u1[:] = S.warm_u(N, seed)
    st.u2[:] = S.warm_u(N, seed + 1)
    rec = {"cfg_" + k: np.asarray(v) for k, v in cfg.items()}
    rec.update(K=K, B=B, d=d, N=N, steps=steps, gamma=gamma, eps=eps)
    rec["state0_u1"] = st.u1.copy()
    rec["state0_u2"] = st.u2.copy()
    for s in range(steps):
        b1, b2 = S.embeddings(B, d, seed * 100 + s)
        ids = S.ids(B, N, seed * 100 + s)
        E1 = S.bf16_to_f32(b1).astype(np.float64)
        E2 = S.bf16_to_f32(b2).astype(np.float64)
        out = O.step(cfg, st, K, E1, E2, ids, gamma, eps, backend="ref")
        rec[f"s{s}_E1bits"] = b1
        rec[f"s{s}_E2bits"] = b2
        rec[f"s{s}_ids"] = ids
        for k, v in out.items():
            rec[f"s{s}_{k}"] = np.asarray(v)
        rec[f"s{s}_tau_after"] = np.asarray(st.tau)
        if st.individual:
            rec[f"s{s}_tau1_after"] = st.tau1.copy()
            rec[f"s{s}_tau2_after"] = st.tau2.copy()
    rec["state_end_u1"] = st.u1.copy()
    rec["state_end_u2"] = st.u2.copy()
    name = f"{var}_K{K}_B{B}_d{d}_s{seed}.npz"
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), name), **rec)
    return name


if __name__ == "__main__":
    for c in CASES:
        print(make(c))
