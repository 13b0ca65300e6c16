"""Shared helpers for the -m gpu parity tests: run the B200 step and the oracle on the same
inputs (bf16 embeddings widened to fp64 for the oracle)."""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_2407_01445_b200 import synthetic as S


def gpu_cfg(ocfg: dict, dim: int, local_batch: int, world: int = 1, rank: int = 0, device: int = 0):
    import paper_2407_01445_b200 as P
    from paper_2407_01445_b200.fastclip import VARIANT_NAMES
    c = P.config_defaults(VARIANT_NAMES[int(ocfg["variant"])], int(ocfg["n_train"]), dim=dim,
                          local_batch=local_batch, world=world, rank=rank, device=device)
    for k in ("tau_init", "tau0", "rho", "tau_lr", "beta1", "beta2", "adam_eps",
              "lr_decay_threshold", "lr_decay_factor"):
        setattr(c, k, float(ocfg[k]))
    for k in ("lr_decay_enabled", "scale_by_tau"):
        setattr(c, k, int(ocfg[k]))
    return c


def to_dev_bf16(bits: np.ndarray, device="cuda"):
    import torch
    return torch.from_numpy(bits.view(np.int16).copy()).to(device).view(torch.bfloat16)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def norm_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run_pair(variant: str, B: int, d: int, N: int, steps: int = 2, gamma: float = 0.6,
             eps: float = 1e-14, seed: int = 0, warm: bool = True, cfg_over=None, checker=None):
    """Runs `steps` K=1 steps on the GPU and in the oracle; returns per-step (gpu, oracle).
    `checker`: the oracle's step function (default: the C restatement, oracle.step; the
    full-size tests pass the vectorised restatement oracle_np.step)."""
    import torch
    import paper_2407_01445_b200 as P
    ocfg = O.default_config(variant, N, **(cfg_over or {}))
    st = O.new_state(ocfg)
    if warm:
        st.u1[:] = S.warm_u(N, seed)
        st.u2[:] = S.warm_u(N, seed + 1)
    step = P.LossStep(gpu_cfg(ocfg, d, B))
    step.load_tables(u1=st.u1, u2=st.u2)
    res = []
    for s in range(steps):
        b1, b2 = S.embeddings(B, d, seed * 1000 + s)
        ids = S.ids(B, N, seed * 1000 + s)
        E1 = S.bf16_to_f32(b1).astype(np.float64)
        E2 = S.bf16_to_f32(b2).astype(np.float64)
        ref = (checker or O.step)(ocfg, st, 1, E1, E2, ids, gamma, eps)
        de1, de2 = step.step(to_dev_bf16(b1), to_dev_bf16(b2), torch.from_numpy(ids).cuda(), gamma, eps)
        sc = step.scalars()
        views = step.local_views()
        got = dict(dE1=de1.cpu().numpy().astype(np.float64), dE2=de2.cpu().numpy().astype(np.float64),
                   loss=sc.loss, gtau=sc.gtau, tau_new=sc.tau, clamps_g=sc.exp_clamps, **views)
        res.append((got, ref))
    tabs = step.tables()
    return res, tabs, st, step
