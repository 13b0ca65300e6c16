"""CPU checks of bench.py's contract helpers (no GPU): the metric string is BASELINE.json's,
the per-rank input slices tile the global batch in rank order (trainer.cpp:231-241), the
workload config names the BASELINE shape, and the roofline traffic lookup finds the committed
ncu summary for every tensor phase."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_metric_matches_baseline():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert json.load(f)["metric"] == bench.METRIC


def test_rank_slices_tile_the_global_batch():
    B, d, N = 64, 16, 10_000
    full = bench.make_inputs(B, d, N, 1, 0, n_sets=2)
    for world in (2, 4):
        parts = [bench.make_inputs(B, d, N, world, r, n_sets=2) for r in range(world)]
        for s in range(2):
            for k in range(3):
                cat = np.concatenate([parts[r][s][k] for r in range(world)])
                np.testing.assert_array_equal(cat, full[s][k])
    ids = full[0][2]
    assert ids.dtype == np.int32 and len(np.unique(ids)) == B and ids.min() >= 0 and ids.max() < N


def test_workload_config_names_the_shape():
    args = argparse.Namespace(variant="fastclip_v3", batch=5120, dim=512, n_train=2_700_000)
    for world in (1, 2, 4, 8):
        cfg = bench.workload_config(args, world)
        assert cfg["global_batch"] == 5120 and cfg["local_batch"] * world == 5120
        assert cfg["dim"] == 512 and cfg["parallelism"].startswith(f"dp{world}")
        assert "workload" in cfg and "l2" in cfg


def test_traffic_lookup_covers_the_tensor_phases():
    for phase in ("pass1_stats", "pass2_q", "grad_gemm"):
        t = bench.ncu_traffic(phase)
        assert t is not None and t["bytes"] > 0 and t["source"].startswith("profiles")
