"""Vectorised numpy restatement of the FastCLIP loss step -- TEST INFRASTRUCTURE ONLY.

The full-size checker: the same arithmetic as oracle/fastclip_oracle.c (fp64, same formulas,
same order of the state updates) written with whole-matrix numpy/BLAS operations, so one step
at the north-star shape (B = 5120, d = 512) takes seconds instead of the serial C oracle's
minutes. Summation order differs from the C restatement (BLAS blocking, pairwise sums), so it
agrees with it to ~1e-12 relative, not bit-exactly; tests/test_oracle.py pins it against the C
oracle (itself bit-exact with the reference TUs) on every variant at K = 1..4.

Citations (reference proj/core/): S = E1 E2^T (losses.cpp:33-41); safe_exp (losses.cpp:22-28);
g (engine.cpp:151-176); u EMA + snapshot (state.cpp:45-71); weights (engine.cpp:28-75,
trainer.cpp:449-491); cotangents (engine.cpp:77-121) in the Q form of SURVEY.md 8(a) row a6:
  P1[a,b] = (w1_a/t1_a) e^{(S_ab - S_aa)/t1_a},  P2[a,b] = (w2_a/t2_a) e^{(S_ba - S_aa)/t2_a},
  Q = P1 + P2^T (zero diagonal),  r = rowsum(P1) + rowsum(P2),
  dE1[L] = c (Q[L,:] E2 - r_L o E2[L]),  dE2[L] = c (Q[:,L]^T E1 - r_L o E1[L]),  c = 1/(Bl(B-1));
dtau sums (engine.cpp:182-204); G_tau (engine.cpp:208-266); exact loss (losses.cpp:103-180);
Adam + projection (optimizers.cpp:65-83); latch (schedules.hpp:55-58).
Only tests/ may import this module.
"""
from __future__ import annotations

import numpy as np

from oracle import (FASTCLIP_V3, ISOGCLR, FASTCLIP_V2, OPENCLIP_MBCL, SOGCLR, FASTCLIP_V1,
                    TableState)

_CLAMP = 60.0   # losses.hpp:22


def _safe_exp(x: np.ndarray) -> tuple[np.ndarray, int]:
    """losses.cpp:22-28 elementwise; returns (exp(min(x, 60)), number of clamped entries)."""
    n = int(np.count_nonzero(x > _CLAMP))
    return np.exp(np.minimum(x, _CLAMP)), n


def _adam_tau(m, v, step, tau, grad, lr, cfg):
    """optimizers.cpp:65-83 (wd = 0, bias correction with step+1, then max(., tau0));
    works elementwise on arrays (v2 per-index state) or on scalars."""
    b1, b2, eps = cfg["beta1"], cfg["beta2"], cfg["adam_eps"]
    if not np.all(np.isfinite(grad)):
        raise RuntimeError("oracle_np: non-finite tau gradient (NumericError)")
    m = b1 * m + (1.0 - b1) * grad
    v = b2 * v + (1.0 - b2) * grad * grad
    c1 = 1.0 - np.power(b1, (step + 1).astype(np.float64) if isinstance(step, np.ndarray) else float(step + 1))
    c2 = 1.0 - np.power(b2, (step + 1).astype(np.float64) if isinstance(step, np.ndarray) else float(step + 1))
    step = step + 1
    r = (m / c1) / (np.sqrt(v / c2) + eps)
    nt = tau - lr * r
    return m, v, step, np.maximum(nt, cfg["tau0"])


def _row_sums(S: np.ndarray, diag: np.ndarray, t: np.ndarray, transpose: bool, block: int = 1024):
    """sum_{j != i} e^{(S_ij - S_ii)/t_i} (or S_ji) and sum_{j != i} -(d/t^2) e^{d/t}, per row i,
    with the clamp count; row-blocked to bound the temporaries."""
    B = S.shape[0]
    se = np.empty(B)
    sd = np.empty(B)
    clamps = 0
    for lo in range(0, B, block):
        hi = min(B, lo + block)
        blk = (S[:, lo:hi].T if transpose else S[lo:hi]) - diag[lo:hi, None]
        tt = t[lo:hi, None]
        e, n = _safe_exp(blk / tt)   # the diagonal entry is 0: never clamped, then excluded
        rows = np.arange(hi - lo)
        e[rows, lo + rows] = 0.0
        clamps += n
        se[lo:hi] = e.sum(axis=1)
        sd[lo:hi] = (-(blk / (tt * tt)) * e).sum(axis=1)
    return se, sd, clamps


def _weighted(S, diag, w, t, transpose, block=1024):
    """P[a, :] = (w_a / t_a) e^{(S_a. - S_aa)/t_a} (S_.a when transpose), diagonal zero."""
    B = S.shape[0]
    P = np.empty((B, B))
    for lo in range(0, B, block):
        hi = min(B, lo + block)
        blk = (S[:, lo:hi].T if transpose else S[lo:hi]) - diag[lo:hi, None]
        e, _ = _safe_exp(blk / t[lo:hi, None])
        rows = np.arange(hi - lo)
        e[rows, lo + rows] = 0.0
        P[lo:hi] = (w[lo:hi] / t[lo:hi])[:, None] * e
    return P


def step(cfg: dict, st: TableState, K: int, E1: np.ndarray, E2: np.ndarray, ids: np.ndarray,
         gamma: float, eps: float) -> dict:
    """oc_step (oracle/fastclip_oracle.c) for K workers, vectorised; updates ``st`` in place and
    returns the same dict as oracle.step."""
    E1 = np.ascontiguousarray(E1, dtype=np.float64)
    E2 = np.ascontiguousarray(E2, dtype=np.float64)
    ids = np.asarray(ids, dtype=np.int64)
    B, d = E1.shape
    if K < 1 or B % K:
        raise ValueError("B must be a multiple of K")
    Bl = B // K
    v = cfg["variant"]
    track_u = v != OPENCLIP_MBCL
    indiv = v in (ISOGCLR, FASTCLIP_V2)
    constant = v in (SOGCLR, FASTCLIP_V1)
    S = E1 @ E2.T                                                   # losses.cpp:40
    diag = np.diagonal(S).copy()
    inv = 1.0 / (B - 1)

    # ---- phase 1: tau^t, g over G \ {i} (engine.cpp:151-176), EMA + snapshot (state.cpp) ----
    t1 = st.tau1[ids].copy() if indiv else np.full(B, st.tau)
    t2 = st.tau2[ids].copy() if indiv else np.full(B, st.tau)
    s1, _, c1 = _row_sums(S, diag, t1, False)
    s2, _, c2 = _row_sums(S, diag, t2, True)
    g1, g2 = s1 * inv, s2 * inv
    out = dict(g1=g1, g2=g2, t1=t1, t2=t2, clamps_g=c1 + c2, gtau1=np.zeros(B), gtau2=np.zeros(B),
               gtau_local=np.zeros(K))
    if track_u:
        if np.any(g1 < 0) or np.any(g2 < 0):
            raise RuntimeError("oracle_np: negative g (domain_error)")
        st.u1[ids] = (1.0 - gamma) * st.u1[ids] + gamma * g1       # state.cpp:52-53
        st.u2[ids] = (1.0 - gamma) * st.u2[ids] + gamma * g2
        u1, u2 = st.u1[ids].copy(), st.u2[ids].copy()              # state.cpp:57-71
    # ---- weights (trainer.cpp:449-491) ----
    if v == OPENCLIP_MBCL:
        u1, u2 = g1.copy(), g2.copy()                               # trainer.cpp:451-457 (tau^t = tau)
        c = 1.0 / (B - 1)
        tt1 = tt2 = np.full(B, st.tau)
        w1, w2 = 1.0 / (c + u1), 1.0 / (c + u2)                     # engine.cpp:65-75
    elif indiv:
        tt1, tt2 = t1, t2
        w1, w2 = (1.0 / (eps + u1)) * t1, (1.0 / (eps + u2)) * t2   # engine.cpp:52-63
    else:
        tt1 = tt2 = np.full(B, st.tau)
        w1, w2 = 1.0 / (eps + u1), 1.0 / (eps + u2)                 # engine.cpp:37-50
        if cfg["scale_by_tau"]:
            w1, w2 = w1 * st.tau, w2 * st.tau
    out.update(u1=u1, u2=u2)

    # ---- cotangents (engine.cpp:77-121) ----
    P1 = _weighted(S, diag, w1, tt1, False)
    P2 = _weighted(S, diag, w2, tt2, True)
    r = P1.sum(axis=1) + P2.sum(axis=1)
    Q = P1
    Q += P2.T
    del P2
    scale = 1.0 / (Bl * (B - 1))
    dE1 = np.empty((B, d))
    dE2 = np.empty((B, d))
    for k in range(K):
        L = slice(k * Bl, (k + 1) * Bl)
        dE1[L] = scale * (Q[L] @ E2 - r[L, None] * E2[L])
        dE2[L] = scale * (Q[:, L].T @ E1 - r[L, None] * E1[L])
    del Q
    out.update(dE1=dE1, dE2=dE2)

    # ---- tau gradients (engine.cpp:182-266) ----
    if not constant:
        _, ds1, _ = _row_sums(S, diag, tt1, False)
        _, ds2, _ = _row_sums(S, diag, tt2, True)
        ds1, ds2 = ds1 * inv, ds2 * inv
        if indiv:
            inv_n = 1.0 / cfg["n_train"]
            out["gtau1"] = inv_n * (np.log(eps + u1) + cfg["rho"] + tt1 * ds1 / (eps + u1))
            out["gtau2"] = inv_n * (np.log(eps + u2) + cfg["rho"] + tt2 * ds2 / (eps + u2))
        else:
            e = 1.0 / (B - 1) if v == OPENCLIP_MBCL else eps
            for k in range(K):
                L = slice(k * Bl, (k + 1) * Bl)
                unscaled = float(np.sum(ds1[L] / (e + u1[L]) + ds2[L] / (e + u2[L]))) / Bl
                if v == FASTCLIP_V3:
                    logs = float(np.sum(np.log(eps + u1[L]) + np.log(eps + u2[L]))) / Bl
                    out["gtau_local"][k] = logs + 2.0 * cfg["rho"] + st.tau * unscaled
                else:
                    out["gtau_local"][k] = unscaled

    # ---- exact loss at tau^t (losses.cpp:126-180) ----
    if v == OPENCLIP_MBCL or not indiv:
        tau_v = np.full(B, st.tau)
        a1, _, _ = _row_sums(S, diag, tau_v, False)
        a2, _, _ = _row_sums(S, diag, tau_v, True)
        gf1, gf2 = a1 / (B - 1), a2 / (B - 1)
        if v == OPENCLIP_MBCL:
            c = 1.0 / (B - 1)
            loss = float(np.sum(np.log(c + gf1) + np.log(c + gf2))) / B
        else:
            loss = st.tau * float(np.sum(np.log(eps + gf1) + np.log(eps + gf2))) / B
            if v == FASTCLIP_V3:
                loss += 2.0 * cfg["rho"] * st.tau
    else:
        a1, _, _ = _row_sums(S, diag, t1, False)
        a2, _, _ = _row_sums(S, diag, t2, True)
        gf1, gf2 = a1 / (B - 1), a2 / (B - 1)
        loss = float(np.sum(t1 * (np.log(eps + gf1) + cfg["rho"]) + t2 * (np.log(eps + gf2) + cfg["rho"]))) / B
    out["loss"] = loss

    # ---- temperature update (trainer.cpp:557-589) ----
    out["gtau"] = 0.0
    out["tau_new"] = st.tau
    if indiv:
        for tn, mn, vn, sn, gn in (("tau1", "m1", "v1", "s1", "gtau1"), ("tau2", "m2", "v2", "s2", "gtau2")):
            m, vv, s, nt = _adam_tau(getattr(st, mn)[ids], getattr(st, vn)[ids], getattr(st, sn)[ids],
                                     getattr(st, tn)[ids], out[gn], cfg["tau_lr"], cfg)
            getattr(st, mn)[ids] = m
            getattr(st, vn)[ids] = vv
            getattr(st, sn)[ids] = s
            getattr(st, tn)[ids] = nt
    elif not constant:
        gt = float(sum(out["gtau_local"][k] for k in range(K))) * (1.0 / K)   # fabric.cpp:73-83
        out["gtau"] = gt
        lr = cfg["tau_lr"]
        if cfg["lr_decay_enabled"]:
            if st.tau < cfg["lr_decay_threshold"]:
                st.latched = 1
            lr *= cfg["lr_decay_factor"] if st.latched else 1.0
        m, vv, s, nt = _adam_tau(st.tau_m, st.tau_v, st.tau_step, st.tau, gt, lr, cfg)
        st.tau_m, st.tau_v, st.tau_step, st.tau = float(m), float(vv), int(s), float(nt)
        out["tau_new"] = st.tau
    return out


def _selftest():   # pragma: no cover -- manual timing
    import time
    import oracle as O
    cfg = O.default_config("fastclip_v3", 100_000)
    st = O.new_state(cfg)
    rng = np.random.default_rng(0)
    B, d = 5120, 512
    E1 = rng.standard_normal((B, d)); E1 /= np.linalg.norm(E1, axis=1, keepdims=True)
    E2 = E1 + rng.standard_normal((B, d)); E2 /= np.linalg.norm(E2, axis=1, keepdims=True)
    ids = rng.choice(100_000, B, replace=False)
    t = time.time()
    step(cfg, st, 1, E1, E2, ids, 0.6, 1e-14)
    print(f"B={B} d={d}: {time.time() - t:.1f} s")


if __name__ == "__main__":
    _selftest()


# ---- the model-side step -- restatement of encoder.cpp:98-177 ----

def tower_forward(kind: int, theta: np.ndarray, x: np.ndarray, d_hidden: int, d_out: int) -> dict:
    """TwoTowerModel::forward (encoder.cpp:98-134): linear z = x W^T + b (:110-113) or tanh-MLP
    (:115-123), then e = z / |z| row-wise (:125-132)."""
    d_in = x.shape[1]
    h = None
    if kind == 0:
        w = theta[:d_out * d_in].reshape(d_out, d_in)
        b = theta[d_out * d_in:d_out * d_in + d_out]
        z = x @ w.T + b
    else:
        H = d_hidden
        w1 = theta[:H * d_in].reshape(H, d_in)
        b1 = theta[H * d_in:H * d_in + H]
        o = H * d_in + H
        w2 = theta[o:o + d_out * H].reshape(d_out, H)
        b2 = theta[o + d_out * H:o + d_out * H + d_out]
        h = np.tanh(x @ w1.T + b1)
        z = h @ w2.T + b2
    zn = np.sqrt(np.sum(z * z, axis=1))
    return dict(x=x, h=h, z=z, e=z / zn[:, None], znorm=zn)


def tower_vjp(kind: int, theta: np.ndarray, tape: dict, cot: np.ndarray) -> np.ndarray:
    """TwoTowerModel::vjp (encoder.cpp:136-177) -> the tower's parameter gradient."""
    e, zn, x, h = tape["e"], tape["znorm"], tape["x"], tape["h"]
    radial = np.sum(e * cot, axis=1, keepdims=True)               # encoder.cpp:153
    cz = (cot - radial * e) / zn[:, None]                          # :154
    d_out, d_in = e.shape[1], x.shape[1]
    if kind == 0:                                                  # :158-163
        return np.concatenate([(cz.T @ x).ravel(), cz.sum(axis=0)])
    H = h.shape[1]
    o = H * d_in + H
    w2 = theta[o:o + d_out * H].reshape(d_out, H)
    gw2 = cz.T @ h                                                 # :172
    gb2 = cz.sum(axis=0)
    ca = (cz @ w2) * (1.0 - h * h)                                 # :174-175
    return np.concatenate([(ca.T @ x).ravel(), ca.sum(axis=0), gw2.ravel(), gb2])
