"""CPU checks of the §8(f) host-side rows against the reference's own code (oracle/_ref, built from
/root/reference): the index stream (BatchPlan, trainer.cpp:206-241) and the synthetic inputs drawn
from the reference's RNG streams (rng.hpp:14-65)."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle as O
import paper_2407_01445_b200 as P
from paper_2407_01445_b200 import synthetic as S


def _ref():
    try:
        return O.lib("ref")
    except FileNotFoundError:
        pytest.skip("reference build (oracle/_ref) absent")


@pytest.mark.parametrize("n,B,seed,world", [(64, 16, 7, 1), (4096, 256, 11, 4), (2_700_000, 5400, 3, 8)])
def test_batch_plan_matches_reference(n, B, seed, world):
    L = _ref()
    plan = P.BatchPlan(n, B, seed)
    assert plan.iters_per_epoch == n // B
    for epoch in (0, 1, 17):
        for it in (0, plan.iters_per_epoch - 1):
            for worker in range(world):
                got = plan.local_batch(epoch, it, worker, world)
                ref = np.empty(B // world, np.int32)
                assert L.ref_batch_plan_local(n, B, seed, epoch, it, worker, world,
                                              ref.ctypes.data_as(C.POINTER(C.c_int))) == 0
                np.testing.assert_array_equal(got, ref)
    perm = plan.permutation(2)
    assert np.array_equal(np.sort(perm), np.arange(n, dtype=np.int32))   # a permutation


def test_batch_plan_errors():
    # trainer.cpp:208-213 (ConfigError), :225 / :233-236 (ShapeError / ConfigError)
    with pytest.raises(P.FastclipError) as e:
        P.BatchPlan(100, 30, 1)
    assert e.value.kind == "ConfigError"
    with pytest.raises(P.FastclipError) as e:
        P.BatchPlan(10, 20, 1)
    assert e.value.kind == "ConfigError"
    plan = P.BatchPlan(120, 12, 1)
    with pytest.raises(P.FastclipError) as e:
        plan.local_batch(0, 10, 0, 1)
    assert e.value.kind == "ShapeError"
    with pytest.raises(P.FastclipError) as e:
        plan.local_batch(0, 0, 0, 5)
    assert e.value.kind == "ConfigError"


def test_synthetic_embeddings_follow_reference_streams():
    # E1 = normalize(Z) with Z from the {0x656d6231} stream's Box-Muller normals, E2 =
    # normalize(E1 + N) with the {0x656d6232} stream, rounded to bf16
    L = _ref()
    seed, B, d = 42, 6, 16
    e1, e2 = S.embeddings(B, d, seed)
    z = np.empty(B * d)
    y = np.empty(B * d)
    L.ref_rng_normals(L.ref_stream_seed2(seed, 0x656d6231, 0, 1), B * d, z.ctypes.data_as(C.POINTER(C.c_double)))
    L.ref_rng_normals(L.ref_stream_seed2(seed, 0x656d6232, 0, 1), B * d, y.ctypes.data_as(C.POINTER(C.c_double)))
    z = z.reshape(B, d)
    z /= np.sqrt(np.sum(z * z, axis=1, keepdims=True))
    w = z + y.reshape(B, d)
    w /= np.sqrt(np.sum(w * w, axis=1, keepdims=True))
    np.testing.assert_array_equal(e1, S.bf16_round(z.astype(np.float32)))
    np.testing.assert_array_equal(e2, S.bf16_round(w.astype(np.float32)))


def test_synthetic_ids_are_distinct_and_follow_reference_stream():
    L = _ref()
    seed, B, N = 5, 300, 1000
    ids = S.ids(B, N, seed)
    assert len(set(ids.tolist())) == B and ids.min() >= 0 and ids.max() < N
    draws = np.empty(B, np.uint64)
    L.ref_rng_below(L.ref_stream_seed2(seed, 0x696473, 0, 1), B, N, draws.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    perm = np.arange(N)
    for i in range(B):   # partial Fisher-Yates with the reference's Rng::below draws
        j = i + int(draws[i])
        perm[i], perm[j] = perm[j], perm[i]
    np.testing.assert_array_equal(ids, perm[:B])
