"""Pins for the CPU oracle (no GPU needed).

The oracle (oracle/bm_oracle.c) is checked against things other than itself:
hand-worked examples (tests/golden/hand_examples.json, each cited), the
eps-net axioms of Def 2.1, an independent brute force built
from scipy distance matrices and sparse products, the LFMIS certificate
(SURVEY §8(c)), closed-form special cases, and the prefix property of the
index-order greedy.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import (balls_of, brute_cover, case_arrays, csr_transpose_ok,
                           edges_from_csr, lfmis_certificate)
from workloads import gen


def test_golden_hand_examples(golden_cases):
    for case in golden_cases:
        X, eps = case_arrays(case)
        c = O.cover(X, case["metric"], eps)
        assert c.landmarks.tolist() == case["landmarks"], case["name"]
        assert balls_of(c.ball_ptr, c.ball_idx) == case["balls"], case["name"]
        assert c.edges.tolist() == case["edges"], case["name"]


def test_spec_range_examples():
    # 1-D {0,1,2,3}, q=0, eps=1.5 -> {0,1}; {0,1}, eps=1 -> {0}
    X = np.array([[0], [1], [2], [3]], dtype=np.float32)
    assert O.range_query(X, "l2", 1.5, 0).tolist() == [0, 1]
    assert O.range_query(X[:2], "l2", 1.0, 0).tolist() == [0]
    # {(0,0),(3,4)}: eps=5 -> {0}; eps=5.001 -> {0,1}
    Y = np.array([[0, 0], [3, 4]], dtype=np.float32)
    assert O.range_query(Y, "l2", 5.0, 0).tolist() == [0]
    assert O.range_query(Y, "l2", 5.001, 0).tolist() == [0, 1]
    # L1 between (1,2) and (4,6) is 7
    Z = np.array([[1, 2], [4, 6]], dtype=np.float32)
    assert O.distance(Z, "l1", 0, 1) == 7.0
    assert O.distance(Z, "l2", 0, 1) == 25.0


def _check_axioms(X, metric, eps, c):
    """Def 2.1: coverage d(x, n) < eps; separation >= eps."""
    D = O.pair_distances
    n = len(X)
    # coverage: every point has a covering landmark at distance < eps
    assert np.all(np.diff(c.pt_ptr) > 0)
    first = c.landmarks[c.pt_lm[c.pt_ptr[:-1]]]
    dist = D(X, metric, np.arange(n), first)
    assert np.all(dist < eps)
    # separation over all landmark pairs
    L = c.L
    if L > 1:
        ii, jj = np.triu_indices(L, 1)
        sep = D(X, metric, c.landmarks[ii], c.landmarks[jj])
        assert np.all(sep >= eps)


@pytest.mark.parametrize("metric", ["l2", "l1", "cos"])
@pytest.mark.parametrize("dtype", ["f32", "i8", "u8"])
@pytest.mark.parametrize("seed", range(6))
def test_brute_force_small(metric, dtype, seed):
    if metric == "cos" and dtype != "f32":
        pytest.skip("cosine is defined on the f32 path only")
    rng = np.random.default_rng([seed, 7])
    n = int(rng.integers(1, 300))
    d = int(rng.integers(1, 9))
    X = gen.random_cloud(n, d, dtype, seed=seed, scale=1.0, lo=-6, hi=6)
    if dtype == "u8":
        X = gen.random_cloud(n, d, dtype, seed=seed, lo=0, hi=12)
    Dm = None
    # choose eps so that balls are neither trivial nor empty; avoid exact ties
    # with the float eps (integers: eps^2 half-integer for L2, half-integer for L1)
    if dtype == "f32":
        eps = {"l2": 0.35 * math.sqrt(d), "l1": 0.3 * d, "cos": 0.05}[metric]
    else:
        eps = {"l2": math.sqrt(2.0 * d + 0.5), "l1": 1.5 * d + 0.5, "cos": 0.1}[metric]
    c = O.cover(X, metric, eps)
    lms, balls, edges, Dm = brute_cover(X, metric, eps)
    # ties in float data would make the two predicates differ only at exactly
    # d == eps; assert none is within 1e-9 relative
    if dtype == "f32":
        assert not np.any(np.abs(Dm - eps) <= 1e-9 * eps)
    assert c.landmarks.tolist() == lms.tolist()
    assert balls_of(c.ball_ptr, c.ball_idx) == balls
    assert c.edges.tolist() == edges.tolist()
    assert csr_transpose_ok(c.L, n, c.ball_ptr, c.ball_idx, c.pt_ptr, c.pt_lm)
    assert lfmis_certificate(c.landmarks, c.pt_ptr, c.pt_lm, n) == []
    _check_axioms(X, metric, eps, c)


def test_c1_full_brute_force():
    w = gen.get("c1")
    X = gen.generate(w)
    c = O.cover(X, w.metric, w.eps)
    lms, balls, edges, _ = brute_cover(X, w.metric, w.eps)
    assert c.landmarks.tolist() == lms.tolist()
    assert balls_of(c.ball_ptr, c.ball_idx) == balls
    assert c.edges.tolist() == edges.tolist()
    assert c.pairs_evaluated == c.L * w.n
    _check_axioms(X, w.metric, w.eps, c)


def test_integer_eps_cut_is_unambiguous():
    """C1: eps^2 = 60.5 and integer squared distances -> no exact tie, and
    d^2 = 60 is not a sum of three squares (reading A10)."""
    sums3 = {a * a + b * b + c * c for a in range(9) for b in range(9) for c in range(9)}
    assert 60 not in sums3 and 59 in sums3 and 61 in sums3
    X = np.array([[0, 0, 0], [7, 3, 1], [7, 3, 2], [5, 5, 3]], dtype=np.int8)  # 59, 62, 59
    c = O.cover(X, "l2", math.sqrt(60.5))
    assert c.landmarks.tolist() == [0, 2]
    assert balls_of(c.ball_ptr, c.ball_idx) == [[0, 1, 3], [1, 2, 3]]


def test_special_cases_closed_form():
    X = gen.random_cloud(200, 5, "f32", seed=3)
    Dm = brute_cover(X, "l2", 1e-9)[3]
    diam = Dm.max()
    c = O.cover(X, "l2", diam * 1.01)               # eps > diameter: one ball = X
    assert c.landmarks.tolist() == [0] and c.M == 200 and c.E == 0
    dmin = Dm[np.triu_indices(200, 1)].min()
    c = O.cover(X, "l2", dmin)                      # eps <= min distance: all singletons
    assert c.landmarks.tolist() == list(range(200))
    assert c.ball_idx.tolist() == list(range(200)) and c.E == 0


def test_prefix_property():
    """Landmarks of X[:m] are landmarks(X) ∩ [0, m) (index-order greedy)."""
    w = gen.get("c2")
    X = gen.generate(w, 6000)
    full = O.cover(X, w.metric, w.eps)
    for m in (1, 17, 1000, 4321):
        pre = O.cover(X[:m], w.metric, w.eps)
        assert pre.landmarks.tolist() == full.landmarks[full.landmarks < m].tolist()


def test_overrides_follow_the_caller():
    """Tie protocol: an override replaces one in-ball decision (hand trace:
    collinear 0..6, eps=2, force point 2 into ball of landmark 0)."""
    X = np.arange(7, dtype=np.float32).reshape(-1, 1)
    c = O.cover(X, "l2", 2.0, overrides=[(2, 0, True)])
    assert c.landmarks.tolist() == [0, 3, 5]
    assert balls_of(c.ball_ptr, c.ball_idx) == [[0, 1, 2], [2, 3, 4], [4, 5, 6]]
    assert c.edges.tolist() == [[0, 1], [1, 2]]


def test_edges_match_sparse_product_and_certificate_c2_prefix():
    w = gen.get("c2")
    X = gen.generate(w, 20000)
    c = O.cover(X, w.metric, w.eps)
    assert c.edges.tolist() == edges_from_csr(c.L, len(X), c.ball_ptr, c.ball_idx).tolist()
    assert lfmis_certificate(c.landmarks, c.pt_ptr, c.pt_lm, len(X)) == []
    assert csr_transpose_ok(c.L, len(X), c.ball_ptr, c.ball_idx, c.pt_ptr, c.pt_lm)


def test_certificate_rejects_wrong_greedy():
    """The certificate itself catches a plausible greedy bug (a dropped
    landmark, an extra landmark)."""
    X = np.arange(7, dtype=np.float32).reshape(-1, 1)
    c = O.cover(X, "l2", 1.5)
    assert lfmis_certificate(c.landmarks, c.pt_ptr, c.pt_lm, 7) == []
    # add a bogus landmark 1 (covered by 0): first(1)=0 <1 but 1 flagged landmark
    bad_lm = np.array([0, 1, 2, 4, 6])
    pt_ptr = np.array([0, 1, 3, 5, 6, 8, 9, 10])
    pt_lm = np.array([0, 0, 1, 1, 2, 2, 2, 3, 3, 4])
    assert lfmis_certificate(bad_lm, pt_ptr, pt_lm, 7) != []


def test_oracle_rejects_invalid_input():
    X = np.zeros((3, 2), dtype=np.float32)
    for eps in (0.0, -1.0, float("nan"), float("inf")):
        with pytest.raises(ValueError):
            O.cover(X, "l2", eps)


# ---------------------------------------------------------------- near-tie band
# oracle.near_tie_band is the gate every float parity test passes through
# (tests/parity.py): a GPU-reported tie is accepted as an override only if it
# lies in |d - eps| <= 1e-6 eps (BASELINE.json north_star).  Pinned here with
# hand-built pairs whose exact distance (50-digit decimal arithmetic on the
# stored fp32 coordinates — not the oracle's fp64 formula) sits at
# eps (1 +- 0.5e-6) (inside) or eps (1 +- 2e-6) (outside), with eps != 1 so a
# slip to d^2, rel*eps^2 or an absolute 1e-6 fails one of them.
def _exact_dist(a, b, metric):
    from decimal import Decimal, getcontext
    getcontext().prec = 50
    x = [Decimal(float(v)) for v in a]   # fp32 -> exact binary value
    y = [Decimal(float(v)) for v in b]
    if metric == "l2":
        return sum((p - q) * (p - q) for p, q in zip(x, y)).sqrt()
    if metric == "l1":
        return sum(abs(p - q) for p, q in zip(x, y))
    dot = sum(p * q for p, q in zip(x, y))
    nx = sum(p * p for p in x).sqrt()
    ny = sum(q * q for q in y).sqrt()
    return 1 - dot / (nx * ny)


def _band_case(metric, eps, rel):
    """Two fp32 points at distance ~ eps (1 + rel) in the given metric."""
    t = 1.0 + rel
    if metric == "l2":      # 3-4-5 triangle scaled: |(3s, 4s)| = 5 s
        s = eps / 5.0 * t
        return np.array([[0.0, 0.0], [3.0 * s, 4.0 * s]], dtype=np.float32)
    if metric == "l1":      # |a| + |b| = eps t, split unevenly over two coordinates
        return np.array([[0.25, -1.0], [0.25 + 0.3 * eps * t, -1.0 - 0.7 * eps * t]],
                        dtype=np.float32)
    # cosine: angle theta with 1 - cos(theta) = eps t, x = (1, 0), y = (cos, sin) * 7
    c = 1.0 - eps * t
    return np.array([[1.0, 0.0], [7.0 * c, 7.0 * math.sqrt(1.0 - c * c)]], dtype=np.float32)


@pytest.mark.parametrize("metric,eps", [("l2", 5.0), ("l2", 0.4), ("l1", 3.0), ("l1", 0.7),
                                        ("cos", 0.5), ("cos", 0.25)])
@pytest.mark.parametrize("rel,inside", [(0.5e-6, True), (-0.5e-6, True), (2e-6, False),
                                        (-2e-6, False), (0.0, True), (5e-5, False)])
def test_near_tie_band_pins(metric, eps, rel, inside):
    from decimal import Decimal
    X = _band_case(metric, eps, rel)
    d = _exact_dist(X[0], X[1], metric)
    dev = abs(d - Decimal(eps)) / Decimal(eps)
    # the construction lands where intended (fp32 storage moves it by < 0.3e-6)
    assert abs(float(dev) - abs(rel)) < 0.3e-6, (metric, eps, rel, float(dev))
    assert (dev <= Decimal("1e-6")) == inside
    got = O.near_tie_band(X, metric, eps, np.array([0]), np.array([1]))
    assert bool(got[0]) == inside, (metric, eps, rel, float(dev))
    # symmetric in the pair order
    assert bool(O.near_tie_band(X, metric, eps, np.array([1]), np.array([0]))[0]) == inside
