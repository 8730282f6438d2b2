"""Pins of the §8(f) oracle (coloring, k-skeleton) against values the paper and
the mathematics fix: hand-worked aggregates, the range condition and the
bounds of Props 2.4 / 2.5, an independent brute force of
the higher simplices from the incidence matrix, and the skeleton's own
structure (k = 1 equals the edge list; every face of a simplex is a simplex,
PAPER.md:77-82)."""
import itertools
import math

import numpy as np
import pytest

from oracle import extensions as X
from oracle import oracle as O
from workloads import gen


# ---------------------------------------------------------------- aggregates
@pytest.mark.parametrize("vals,agg,alpha,want", [
    ([1, 2, 3], "mean", 0.0, 2.0),
    ([1, 2, 3], "median", 0.0, 2.0),
    ([1, 2, 3, 4], "median", 0.0, 2.5),          # even size: mean of the central pair
    ([4, 1, 3, 2], "median", 0.0, 2.5),          # order does not matter
    ([1, 2, 3, 100], "trimmed", 0.25, 2.5),      # drop floor(0.25*4)=1 at each end
    ([1, 2, 3, 100], "trimmed", 0.2, 26.5),      # floor(0.8)=0: plain mean
    ([5, -1, 7], "min", 0.0, -1.0),
    ([5, -1, 7], "max", 0.0, 7.0),
    ([0, 0, 1], "mode", 0.0, 0.0),               # labels {A, A, B} -> A
    ([2, 2, 1, 1], "mode", 0.0, 1.0),            # tie -> smallest value
    ([1, 3], "variance", 0.0, 1.0),              # population variance
    ([2, 7, 4], "range", 0.0, 5.0),
])
def test_aggregate_hand(vals, agg, alpha, want):
    assert X.aggregate(np.array(vals, dtype=np.float64), agg, alpha) == want


def test_variance_and_range_break_the_range_condition():
    """variance and range need not lie between the ball's min and max."""
    v = np.array([0.0, 10.0])
    assert X.aggregate(v, "variance") > v.max()
    w = np.array([10.0, 11.0])
    assert X.aggregate(w, "range") < w.min()


def _cloud(seed, n=400, d=3):
    rng = np.random.default_rng([seed, 5])
    return rng.normal(size=(n, d)).astype(np.float32)


@pytest.mark.parametrize("seed", range(6))
def test_props_2_4_and_2_5(seed):
    """f = first coordinate is 1-Lipschitz under L2 (k = 1).  For aggregators
    with the range condition: min <= c <= max over the ball;
    |c(l_i) - f(l_i)| < k eps (every ball point is within eps of its centre);
    every value in the ball is within 2 k eps of the colour (the ball's
    diameter is 2 eps); adjacent colours differ by less than 4 k eps.  These
    are the corrected bounds of Props 2.4 / 2.5 (reading C5; the
    literal k eps / 2 k eps fail, see the next test)."""
    Xp = _cloud(seed)
    eps = 0.6
    c = O.cover(Xp, "l2", eps)
    f = Xp[:, 0].astype(np.float64)
    for agg in ("mean", "median", "trimmed", "min", "max"):
        col = X.color(c.ball_ptr, c.ball_idx, f, agg, 0.2)
        for j in range(c.L):
            fv = f[c.ball_idx[c.ball_ptr[j]:c.ball_ptr[j + 1]]]
            assert fv.min() <= col[j] <= fv.max()                 # range condition
            assert abs(col[j] - f[c.landmarks[j]]) < eps          # centre: k eps
            assert np.abs(fv - col[j]).max() < 2 * eps            # any ball point: 2 k eps
        for a, b in c.edges.reshape(-1, 2):
            assert abs(col[a] - col[b]) < 4 * eps                 # adjacent: 4 k eps


def test_prop_2_4_literal_bound_counterexample():
    """PAPER.md:151-163 claims max_x |f(x) - c(l_i)| <= k eps; its proof uses
    d(x, x_i) < eps for two arbitrary ball points, but two points of one ball
    can be 2 eps - delta apart.  1-D, f = identity (k = 1), eps = 1: the
    greedy picks 0, ball {-0.9, 0, 0.9}; colour = min = -0.9 and f(0.9) is
    1.8 > k eps away."""
    pts = np.array([[0.0], [-0.9], [0.9]], dtype=np.float32)
    c = O.cover(pts, "l2", 1.0)
    f = pts[:, 0].astype(np.float64)
    col = X.color(c.ball_ptr, c.ball_idx, f, "min")
    assert c.L == 1 and col[0] == np.float32(-0.9)
    assert abs(f[2] - col[0]) > 1.0              # > k eps: the literal statement fails
    assert abs(f[2] - col[0]) < 2.0              # < 2 k eps: the corrected bound holds


def test_constant_function_colours():
    Xp = _cloud(9)
    c = O.cover(Xp, "l2", 0.5)
    f = np.full(len(Xp), 3.25)
    for agg in ("mean", "median", "trimmed", "min", "max", "mode"):
        assert np.all(X.color(c.ball_ptr, c.ball_idx, f, agg, 0.1) == 3.25)
    assert np.all(X.color(c.ball_ptr, c.ball_idx, f, "variance") == 0.0)
    assert np.all(X.color(c.ball_ptr, c.ball_idx, f, "range") == 0.0)


# ---------------------------------------------------------------- skeleton
def _brute_simplices(c, n, k):
    """Independent: (k+1)-sets of landmarks whose balls share a data point,
    from the dense point x landmark incidence matrix."""
    B = np.zeros((n, c.L), dtype=bool)
    for j in range(c.L):
        B[c.ball_idx[c.ball_ptr[j]:c.ball_ptr[j + 1]], j] = True
    out = [s for s in itertools.combinations(range(c.L), k + 1) if B[:, list(s)].all(axis=1).any()]
    return np.array(out, dtype=np.int64).reshape(-1, k + 1)


def test_skeleton_grid_hand():
    """3x3 grid at eps^2 = 2.5 (tests/golden): landmarks (0,2,6,8), the centre
    lies in all four balls, so every triple of landmarks is a triangle and the
    4-set is a 3-simplex."""
    pts = np.array([[x, y] for y in range(3) for x in range(3)], dtype=np.float32)
    c = O.cover(pts, "l2", math.sqrt(2.5))
    assert c.landmarks.tolist() == [0, 2, 6, 8]
    tri = X.skeleton(c.pt_ptr, c.pt_lm, 2)
    assert tri.tolist() == [list(t) for t in itertools.combinations(range(4), 3)]
    assert X.skeleton(c.pt_ptr, c.pt_lm, 3).tolist() == [[0, 1, 2, 3]]


@pytest.mark.parametrize("seed", range(5))
def test_skeleton_brute_force_and_closure(seed):
    Xp = _cloud(seed, n=300, d=2)
    c = O.cover(Xp, "l2", 0.45)
    e1 = X.skeleton(c.pt_ptr, c.pt_lm, 1)
    assert np.array_equal(e1, c.edges.reshape(-1, 2))                 # k = 1 is the graph
    for k in (2, 3):
        s = X.skeleton(c.pt_ptr, c.pt_lm, k)
        assert np.array_equal(s, _brute_simplices(c, len(Xp), k))
        lower = {tuple(r) for r in X.skeleton(c.pt_ptr, c.pt_lm, k - 1)}
        for simplex in s:                                            # downward closed
            for face in itertools.combinations(simplex, k):
                assert tuple(face) in lower


def test_c1_skeleton_counts_consistent():
    w = gen.get("c1")
    Xp = gen.generate(w)
    c = O.cover(Xp, w.metric, w.eps)
    t = X.skeleton(c.pt_ptr, c.pt_lm, 2)
    # every triangle is witnessed by a point whose row contains it
    rows = [set(c.pt_lm[c.pt_ptr[p]:c.pt_ptr[p + 1]].tolist()) for p in range(len(Xp))]
    for tri in t[:200]:
        assert any(set(tri.tolist()) <= r for r in rows)


# ---------------------------------------------------------------- FPS (NEXT-2)
def test_fps_spec_example():
    """1-D {0,1,2,3}, eps 1.5, start 0 -> (0, 3)."""
    pts = np.array([[0.0], [1.0], [2.0], [3.0]], dtype=np.float32)
    assert O.fps(pts, "l2", 1.5).tolist() == [0, 3]


def test_fps_hand_collinear():
    """0..6 unit spacing, eps 2.5: 0, then 6 (distance 6), then 3 (distance 3);
    the remaining max-min distance is 1 < 2.5."""
    pts = np.arange(7, dtype=np.float32).reshape(-1, 1)
    assert O.fps(pts, "l2", 2.5).tolist() == [0, 6, 3]
    assert O.fps(pts, "l1", 2.5).tolist() == [0, 6, 3]


def test_fps_ge_reading():
    """Reading F1: a point at exactly eps from the landmarks is added
    (with the paper's literal '>' it would stay uncovered by the open ball)."""
    pts = np.array([[0.0], [1.5]], dtype=np.float32)
    assert O.fps(pts, "l2", 1.5).tolist() == [0, 1]
    c = O.cover(pts, "l2", 1.5, landmarks=[0, 1])
    assert c.ball_idx.tolist() == [0, 1]                 # each point in its own ball only


def _brute_fps_int(Xi, eps):
    """Independent FPS on integer data: exact int64 squared distances, numpy argmax."""
    Xl = Xi.astype(np.int64)
    d2 = ((Xl[:, None, :] - Xl[None, :, :]) ** 2).sum(-1)
    mind = d2[0].copy()
    seq = [0]
    while True:
        b = int(np.argmax(mind))                   # first maximum = lowest index
        if not mind[b] >= eps * eps:
            break
        seq.append(b)
        mind = np.minimum(mind, d2[b])
    return seq


@pytest.mark.parametrize("seed", range(5))
def test_fps_brute_force_and_axioms(seed):
    rng = np.random.default_rng([seed, 9])
    Xi = rng.integers(-30, 30, size=(300, 3)).astype(np.int8)
    eps = float(np.sqrt(150.5))
    seq = O.fps(Xi, "l2", eps)
    assert seq.tolist() == _brute_fps_int(Xi, eps)
    from tests.helpers import brute_distance_matrix
    for metric, e in (("l2", 0.7), ("l1", 1.1), ("cos", 0.08)):
        Xf = rng.normal(size=(250, 4)).astype(np.float32)
        s = O.fps(Xf, metric, e)
        D = brute_distance_matrix(Xf, metric)
        assert len(set(s.tolist())) == len(s)
        assert (D[:, s].min(axis=1) < e).all()                     # coverage (Def 2.1)
        sub = D[np.ix_(s, s)] + np.eye(len(s)) * 1e9
        assert (sub >= e - 1e-12).all()                            # separation (Def 2.1)
        c = O.cover(Xf, metric, e, landmarks=np.sort(s))           # cover of the FPS set
        for j, lm in enumerate(np.sort(s)):
            assert c.ball_idx[c.ball_ptr[j]:c.ball_ptr[j + 1]].tolist() == \
                np.nonzero(D[:, lm] < e)[0].tolist()
