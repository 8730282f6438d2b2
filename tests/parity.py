"""GPU-vs-oracle comparator (tie-aware, SURVEY §8(c) parity rules).

Integer workloads: every array bit-exact.  Float workloads: the GPU reports
its near ties (|d_fp64 - eps| <= 1e-6 eps); each one is verified to be inside
that band by the ORACLE's own fp64 distance, fed back to the oracle as an
override, and then every array must be identical.  The number of near ties
must be < 1e-6 of the N*L pairs evaluated (BASELINE.json north_star).
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def gpu_arrays(cov) -> dict:
    a = cov.numpy()
    return {k: np.asarray(v, dtype=np.int64) for k, v in a.items()}


def compare(X: np.ndarray, metric: str, eps: float, cov, *, float_path: bool,
            oracle_result=None, tie_rate_limit: bool = False, landmarks=None) -> dict:
    """landmarks: compare against the oracle's cover of this ascending
    landmark list (the FPS selection) instead of the greedy's.
    tie_rate_limit: enforce north_star's "< 1e-6 of the pairs evaluated" —
    a property of the BASELINE workloads, not of arbitrary random test clouds."""
    g = gpu_arrays(cov)
    overrides = []
    if float_path and len(cov.near_ties):
        assert cov.stats.n_near_ties == len(cov.near_ties), "near-tie list truncated"
        p, q, v = cov.near_ties[:, 0], cov.near_ties[:, 1], cov.near_ties[:, 2]
        band = O.near_tie_band(X, metric, eps, p, q)
        assert band.all(), "GPU reported a near tie outside the 1e-6*eps band"
        overrides = list(zip(p.tolist(), q.tolist(), (v != 0).tolist()))
    if not float_path:
        assert cov.stats.n_near_ties == 0
    n = X.shape[0]
    if oracle_result is None or overrides:
        oracle_result = O.cover(X, metric, eps, overrides=overrides, landmarks=landmarks)
    o = oracle_result
    assert g["landmarks"].tolist() == o.landmarks.tolist(), "landmarks differ"
    assert np.array_equal(g["ball_ptr"], o.ball_ptr), "ball_ptr differs"
    assert np.array_equal(g["ball_idx"], o.ball_idx), "ball_idx differs"
    assert np.array_equal(g["pt_ptr"], o.pt_ptr), "pt_ptr differs"
    assert np.array_equal(g["pt_lm"], o.pt_lm), "pt_lm differs"
    assert np.array_equal(g["edges"].reshape(-1, 2), o.edges.reshape(-1, 2)), "edges differ"
    pairs = n * o.L
    assert cov.stats.n_pair_evals == pairs
    if float_path and tie_rate_limit:
        assert cov.stats.n_near_ties < max(1.0, 1e-6 * pairs), "too many near ties"
    return {"L": o.L, "M": o.M, "E": o.E, "near_ties": int(cov.stats.n_near_ties),
            "band": int(cov.stats.n_band_pairs)}
