"""Synthetic inputs for the loss step, shared by bench, tests and smoke.

Embeddings: E1 = normalize(Z), E2 = normalize(E1 + sigma * N(0, I)) (mean s_ii ~ 0.7 at
sigma = 1), then rounded to bf16 WITHOUT renormalising; the oracle is fed the exact bf16
values widened to fp64. ids: B distinct table indices in [0, N). Tables: cold (u = 0,
state.cpp:42-43) or warm (log10 u ~ U[-8, 0], the paper's u percentiles).
"""
from __future__ import annotations

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even), returned as the uint16 bit patterns."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((b >> 16) & 1) + np.uint32(0x7FFF)
    return ((b + rounding) >> 16).astype(np.uint16)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def embeddings(B: int, d: int, seed: int = 0, sigma: float = 1.0):
    """Returns (E1_bits, E2_bits) as uint16 [B, d] bf16 patterns."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((B, d))
    e1 = z / np.linalg.norm(z, axis=1, keepdims=True)
    n = rng.standard_normal((B, d))
    e2 = e1 + sigma * n
    e2 = e2 / np.linalg.norm(e2, axis=1, keepdims=True)
    return bf16_round(e1.astype(np.float32)), bf16_round(e2.astype(np.float32))


def ids(B: int, N: int, seed: int = 0) -> np.ndarray:
    """B distinct ids in [0, N) (partial Fisher-Yates), int32."""
    rng = np.random.default_rng(seed + 7919)
    if N <= 4 * B:
        return rng.permutation(N)[:B].astype(np.int32)
    out = np.unique(rng.integers(0, N, size=2 * B))
    while out.size < B:
        out = np.unique(np.concatenate([out, rng.integers(0, N, size=B)]))
    rng.shuffle(out)
    return out[:B].astype(np.int32)


def warm_u(n: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed + 31337)
    return 10.0 ** rng.uniform(-8.0, 0.0, size=n)
