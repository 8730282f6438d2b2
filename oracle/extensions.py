"""Oracle for the rows SURVEY §8(f) marks "next": coloring (NEXT-1) and the
k-skeleton (NEXT-3).  Plain per-ball / per-point Python + numpy, fp64.

TEST INFRASTRUCTURE ONLY — only ``tests/`` (and ``__graft_entry__.smoke()`` /
``bench.py``'s oracle legs) may import this module.  It shares no code with
the CUDA product path; its inputs are the oracle's own cover (``oracle.cover``)
or plain arrays.

Coloring (PAPER.md:125-133 [§2.3]): for landmark l_i with ball
X_i = X ∩ B(l_i, eps), c(l_i) = aggregate of f over X_i.  The paper names the
mean, median, trimmed mean, minimum, maximum (all satisfying
the range condition of Prop 2.4), variance and range (which do not),
and the mode / majority vote for labels.  Where the paper is silent
(readings C1-C4): median of an even-size ball = mean of the two
central order statistics; trimmed mean(alpha) drops floor(alpha m) smallest
and largest values; variance is the population variance (divide by m); mode
ties go to the smallest value.

k-skeleton (Def 2.2): a set of k+1 landmarks is a simplex iff
some data point lies in all of their balls (∩ B ∩ X ≠ ∅).  Written here as
the per-point enumeration of the (k+1)-subsets of each point's landmark set,
then sort + unique.
"""
from __future__ import annotations

import itertools

import numpy as np

AGGS = ("mean", "median", "trimmed", "min", "max", "mode", "variance", "range")


def _ball(ball_ptr, ball_idx, j):
    return np.asarray(ball_idx[ball_ptr[j]:ball_ptr[j + 1]], dtype=np.int64)


def aggregate(v: np.ndarray, agg: str, alpha: float = 0.1) -> float:
    """One ball's aggregate (v: the ball's values, fp64)."""
    v = np.asarray(v, dtype=np.float64)
    m = len(v)
    if m == 0:
        return float("nan")
    if agg == "mean":
        return float(v.sum() / m)
    if agg == "median":                     # P:167; even size: mean of the two central values
        s = np.sort(v)
        return float(s[(m - 1) // 2]) if m % 2 == 1 else float((s[m // 2 - 1] + s[m // 2]) / 2.0)
    if agg == "trimmed":                    # P:167; drop floor(alpha m) at each end
        s = np.sort(v)
        t = int(np.floor(alpha * m))
        core = s[t:m - t]
        return float(core.sum() / len(core))
    if agg == "min":
        return float(v.min())
    if agg == "max":
        return float(v.max())
    if agg == "mode":                       # P:187; ties -> smallest value
        vals, counts = np.unique(v, return_counts=True)
        return float(vals[np.argmax(counts)])   # np.unique is ascending, argmax takes the first
    if agg == "variance":                   # P:167 (population variance)
        mu = v.sum() / m
        return float(((v - mu) ** 2).sum() / m)
    if agg == "range":
        return float(v.max() - v.min())
    raise ValueError(agg)


def color(ball_ptr, ball_idx, values, agg: str, alpha: float = 0.1) -> np.ndarray:
    """c(l_j) for every landmark j of a cover (landmark-major CSR)."""
    values = np.asarray(values, dtype=np.float64)
    L = len(ball_ptr) - 1
    return np.array([aggregate(values[_ball(ball_ptr, ball_idx, j)], agg, alpha)
                     for j in range(L)], dtype=np.float64)


def skeleton(pt_ptr, pt_lm, k: int) -> np.ndarray:
    """All k-simplices (k+1 landmark positions, ascending, lexicographic) of
    the nerve: every (k+1)-subset of some point's landmark set (Def 2.2)."""
    out = set()
    n = len(pt_ptr) - 1
    for p in range(n):
        row = [int(x) for x in pt_lm[pt_ptr[p]:pt_ptr[p + 1]]]
        for c in itertools.combinations(sorted(row), k + 1):
            out.add(c)
    return np.array(sorted(out), dtype=np.int64).reshape(-1, k + 1)
