"""Synthetic inputs for the loss step, shared by bench, tests and smoke; drawn
from the reference's deterministic RNG streams (rng.hpp:14-65) through the library's host-side
generator (csrc/batch_plan.cu), so a seed names the same inputs on every machine.

Embeddings: E1 = normalize(Z), E2 = normalize(E1 + sigma * N(0, I)) (mean s_ii ~ 0.7 at
sigma = 1), then rounded to bf16 WITHOUT renormalising; the oracle is fed the exact bf16
values widened to fp64. ids: B distinct table indices in [0, N). Tables: cold (u = 0,
state.cpp:42-43) or warm (log10 u ~ U[-8, 0], the paper's u percentiles).
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even), returned as the uint16 bit patterns."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((b >> 16) & 1) + np.uint32(0x7FFF)
    return ((b + rounding) >> 16).astype(np.uint16)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def embeddings(B: int, d: int, seed: int = 0, sigma: float = 1.0):
    """Returns (E1_bits, E2_bits) as uint16 [B, d] bf16 patterns, drawn from the seed's rng.hpp
    streams (fc_synthetic_embeddings: std::mt19937_64 behind the reference's splitmix64 stream
    ids, two-uniform Box-Muller)."""
    e1 = np.empty((B, d), np.uint16)
    e2 = np.empty((B, d), np.uint16)
    rc = _lib().fc_synthetic_embeddings(int(seed), int(B), int(d), float(sigma), e1.ctypes.data_as(_U16P),
                                        e2.ctypes.data_as(_U16P))
    if rc:
        raise ValueError(f"fc_synthetic_embeddings failed ({rc})")
    return e1, e2


def ids(B: int, N: int, seed: int = 0) -> np.ndarray:
    """B distinct ids in [0, N), int32: a partial Fisher-Yates with the reference's Rng::below."""
    out = np.empty(B, np.int32)
    rc = _lib().fc_synthetic_ids(int(seed), int(B), int(N), out.ctypes.data_as(_I32P))
    if rc:
        raise ValueError(f"fc_synthetic_ids failed ({rc})")
    return out


def warm_u(n: int, seed: int = 0) -> np.ndarray:
    """A warm u table: log10 u ~ U[-8, 0] from the seed's rng stream."""
    out = np.empty(n, np.float64)
    rc = _lib().fc_synthetic_warm_u(int(seed), int(n), out.ctypes.data_as(_F64P))
    if rc:
        raise ValueError(f"fc_synthetic_warm_u failed ({rc})")
    return out


_U16P = C.POINTER(C.c_uint16)
_I32P = C.POINTER(C.c_int32)
_F64P = C.POINTER(C.c_double)


_SYN = None


def _lib():
    # the in-tree build (not an FC_LIB_PATH override: an A/B against an older build still draws
    # the same inputs)
    global _SYN
    if _SYN is None:
        from . import build as _build
        _SYN = C.CDLL(_build.build())
    L = _SYN
    if not getattr(L, "_synthetic_typed", False):
        L.fc_synthetic_embeddings.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_double, _U16P, _U16P]
        L.fc_synthetic_ids.argtypes = [C.c_uint64, C.c_int32, C.c_int64, _I32P]
        L.fc_synthetic_warm_u.argtypes = [C.c_uint64, C.c_int64, _F64P]
        L._synthetic_typed = True
    return L
