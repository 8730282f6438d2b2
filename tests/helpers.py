"""Shared test helpers: case decoding, independent brute force, certificates.

Nothing here is on the product path.  The brute-force routines deliberately use
*different* machinery from the oracle (scipy ``cdist`` distance matrices and
``scipy.sparse`` products) so that they pin the oracle rather than retype it.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
from scipy.spatial.distance import cdist

NP_DTYPES = {"f32": np.float32, "i8": np.int8, "u8": np.uint8}


def case_arrays(case):
    X = np.asarray(case["points"], dtype=NP_DTYPES[case["dtype"]])
    eps = math.sqrt(case["eps2"]) if "eps2" in case else float(case["eps"])
    return X, eps


def balls_of(ball_ptr, ball_idx):
    return [ball_idx[ball_ptr[j]:ball_ptr[j + 1]].tolist() for j in range(len(ball_ptr) - 1)]


def brute_distance_matrix(X: np.ndarray, metric: str) -> np.ndarray:
    """All-pairs fp64 distances via scipy (independent of the oracle)."""
    Xd = X.astype(np.float64)
    if metric == "l2":
        return cdist(Xd, Xd, "euclidean")
    if metric == "l1":
        return cdist(Xd, Xd, "cityblock")
    if metric == "cos":
        nrm = np.linalg.norm(Xd, axis=1)
        D = np.ones((len(Xd), len(Xd)))
        nz = nrm > 0
        D[np.ix_(nz, nz)] = cdist(Xd[nz], Xd[nz], "cosine")
        z = ~nz
        D[np.ix_(z, z)] = 0.0
        return D
    raise ValueError(metric)


def brute_cover(X: np.ndarray, metric: str, eps: float):
    """Brute-force cover from a full distance matrix: LFMIS of the graph
    'd < eps' in index order, membership from matrix rows, edges from the
    sparse product B^T B (off-diagonal nonzero pattern)."""
    D = brute_distance_matrix(X, metric)
    A = D < eps
    n = len(X)
    covered = np.zeros(n, dtype=bool)
    lms = []
    for i in range(n):
        if not covered[i]:
            lms.append(i)
            covered |= A[i]
    lms = np.array(lms, dtype=np.int64)
    B = sp.csr_matrix(A[:, lms].astype(np.int64))       # n x L incidence
    G = (B.T @ B).tocoo()
    edges = sorted({(int(a), int(b)) for a, b in zip(G.row, G.col) if a < b})
    balls = [np.nonzero(A[:, l])[0].tolist() for l in lms]
    return lms, balls, np.array(edges, dtype=np.int64).reshape(-1, 2), D


def lfmis_certificate(landmarks, pt_ptr, pt_lm, n):
    """SURVEY §8(c) certificate: for every point i, pt_lm[i] is non-empty and
    first(i) = landmarks[pt_lm[i][0]] <= i with equality iff i is a landmark.
    Returns a list of violations (empty == certified)."""
    landmarks = np.asarray(landmarks)
    pt_ptr = np.asarray(pt_ptr)
    pt_lm = np.asarray(pt_lm)
    is_lm = np.zeros(n, dtype=bool)
    is_lm[landmarks] = True
    cnt = np.diff(pt_ptr)
    bad = []
    empty = np.nonzero(cnt == 0)[0]
    if len(empty):
        bad.append(("uncovered", empty[:10].tolist()))
    nz = np.nonzero(cnt > 0)[0]
    first = landmarks[pt_lm[pt_ptr[nz]]]
    viol = nz[(first > nz) | ((first == nz) != is_lm[nz])]
    if len(viol):
        bad.append(("first", viol[:10].tolist()))
    return bad


def csr_transpose_ok(L, n, ball_ptr, ball_idx, pt_ptr, pt_lm) -> bool:
    """The point-major CSR is exactly the transpose of the landmark-major one."""
    a = sp.csr_matrix((np.ones(len(ball_idx)), np.asarray(ball_idx), np.asarray(ball_ptr)),
                      shape=(L, n))
    b = sp.csr_matrix((np.ones(len(pt_lm)), np.asarray(pt_lm), np.asarray(pt_ptr)),
                      shape=(n, L))
    return (a.T != b).nnz == 0


def edges_from_csr(L, n, ball_ptr, ball_idx):
    """Edges as the off-diagonal pattern of B B^T with B the L x n incidence
    (scipy.sparse; independent of pair enumeration)."""
    B = sp.csr_matrix((np.ones(len(ball_idx), dtype=np.int64), np.asarray(ball_idx),
                       np.asarray(ball_ptr)), shape=(L, n))
    G = (B @ B.T).tocoo()
    m = G.row < G.col
    e = np.stack([G.row[m], G.col[m]], axis=1).astype(np.int64)
    if len(e) == 0:
        return e.reshape(0, 2)
    order = np.lexsort((e[:, 1], e[:, 0]))
    return e[order]


def fullsize_validity(X, metric, eps, a, near_ties, *, seed=0, n_pairs=10_000_000,
                      n_rows=100, n_cols=40, n_edge_pts=20_000, n_edges=20_000,
                      chunk=5_000_000):
    """Oracle-independent-of-size validity of a GPU cover at full scale
    (SURVEY §8(c) "What pins each part"):

    1. the LFMIS certificate (coverage + first(i) <= i, = iff landmark), which
       given a correct membership proves the landmark list is the greedy's;
    2. the point-major CSR is exactly the transpose of the landmark-major one;
    3. every reported membership (p, l) is in the ball by the oracle's own fp64
       predicate (oracle.pair_inball), up to reported near ties;
    4. >= n_pairs uniformly sampled (point, landmark) pairs decided the same
       way by the GPU (CSR lookup) and the oracle;
    5. complete rows / columns: for n_rows random points every landmark, and
       for n_cols random landmarks every point, re-decided by the oracle
       (catches a missing membership that uniform sampling would miss);
    6. edges: for sampled points every pair of their landmarks is an edge,
       and sampled edges have a witness point in both balls (sorted-list
       intersection of the two balls).
    Disagreements are allowed only on pairs the GPU reported as near ties
    that the oracle places inside the 1e-6*eps band.  Returns a report dict;
    raises AssertionError on any violation."""
    from oracle import oracle as O
    rng = np.random.default_rng([seed, 0xF5])
    n = X.shape[0]
    lms = np.asarray(a["landmarks"], dtype=np.int64)
    L = len(lms)
    ball_ptr = np.asarray(a["ball_ptr"], dtype=np.int64)
    ball_idx = np.asarray(a["ball_idx"], dtype=np.int64)
    pt_ptr = np.asarray(a["pt_ptr"], dtype=np.int64)
    pt_lm = np.asarray(a["pt_lm"], dtype=np.int64)
    edges = np.asarray(a["edges"], dtype=np.int64).reshape(-1, 2)
    M = len(pt_lm)
    rep = {"n": int(n), "L": int(L), "M": int(M), "E": int(len(edges))}
    ties = set()
    if len(near_ties):
        nt = np.asarray(near_ties, dtype=np.int64)
        band = O.near_tie_band(X, metric, eps, nt[:, 0], nt[:, 1])
        assert band.all(), "GPU near tie outside the oracle's band"
        ties = set(zip(nt[:, 0].tolist(), nt[:, 1].tolist()))
    rep["near_ties"] = len(ties)
    assert len(ties) < max(1.0, 1e-6 * n * L), "too many near ties"

    def agree(p, j, gpu_in):
        """Oracle decision of (p, landmark position j) vs the GPU's; returns #checked."""
        q = lms[j]
        o = O.pair_inball(X, metric, eps, p, q)
        bad = np.nonzero(o != gpu_in)[0]
        for k in bad.tolist():
            assert (int(p[k]), int(q[k])) in ties, (
                f"pair (point {int(p[k])}, landmark {int(q[k])}): GPU {bool(gpu_in[k])}, "
                f"oracle {bool(o[k])}, not a reported near tie")
        return len(p), len(bad)

    # 1. certificate
    bad = lfmis_certificate(lms, pt_ptr, pt_lm, n)
    assert bad == [], f"LFMIS certificate violated: {bad}"
    assert np.all(np.diff(lms) > 0) and lms[0] == 0
    rep["certificate"] = "ok"
    # 2. transpose: the landmark-major CSR regrouped by point equals pt_lm
    cnt = np.diff(ball_ptr)
    assert cnt.sum() == M and pt_ptr[-1] == M and ball_ptr[-1] == M
    lm_of = np.repeat(np.arange(L, dtype=np.int64), cnt)
    key_lm = ball_idx * L + lm_of                      # (point, position) from the balls
    key_pt = np.repeat(np.arange(n, dtype=np.int64), np.diff(pt_ptr)) * L + pt_lm
    assert np.all(np.diff(key_pt) > 0), "pt_lm not ascending within points"
    assert np.all(np.diff(ball_idx)[np.diff(lm_of) == 0] > 0), "balls not ascending"
    assert np.array_equal(np.sort(key_lm), key_pt), "CSR transpose mismatch"
    del key_lm, lm_of
    rep["transpose"] = "ok"

    def gpu_member(p, j):
        k = p * L + j
        i = np.searchsorted(key_pt, k)
        i = np.minimum(i, M - 1)
        return key_pt[i] == k

    # 3. every reported membership is in the ball
    pts = np.repeat(np.arange(n, dtype=np.int64), np.diff(pt_ptr))
    checked = disagree = 0
    for s in range(0, M, chunk):
        c, b = agree(pts[s:s + chunk], pt_lm[s:s + chunk], np.ones(min(chunk, M - s), bool))
        checked += c
        disagree += b
    del pts
    rep["members_checked"] = checked
    # 4. uniform pairs
    for s in range(0, n_pairs, chunk):
        m = min(chunk, n_pairs - s)
        p = rng.integers(0, n, m)
        j = rng.integers(0, L, m)
        c, b = agree(p, j, gpu_member(p, j))
        checked += c
        disagree += b
    rep["uniform_pairs"] = int(n_pairs)
    # 5. complete rows and columns
    rows = rng.choice(n, size=min(n_rows, n), replace=False)
    for p0 in rows.tolist():
        j = np.arange(L, dtype=np.int64)
        p = np.full(L, p0, dtype=np.int64)
        c, b = agree(p, j, gpu_member(p, j))
        checked += c
        disagree += b
    cols = rng.choice(L, size=min(n_cols, L), replace=False)
    for j0 in cols.tolist():
        p = np.arange(n, dtype=np.int64)
        j = np.full(n, j0, dtype=np.int64)
        c, b = agree(p, j, gpu_member(p, j))
        checked += c
        disagree += b
    rep["full_rows"] = int(len(rows))
    rep["full_cols"] = int(len(cols))
    rep["pairs_rechecked"] = int(checked)
    rep["tie_disagreements"] = int(disagree)
    # 6. edges
    ekey = edges[:, 0] * L + edges[:, 1]
    assert np.all(np.diff(ekey) > 0), "edges not sorted / unique"
    assert np.all(edges[:, 0] < edges[:, 1]) if len(edges) else True
    sp_ = rng.choice(n, size=min(n_edge_pts, n), replace=False)
    need = []
    for p0 in sp_.tolist():
        row = pt_lm[pt_ptr[p0]:pt_ptr[p0 + 1]]
        if len(row) > 1:
            ii, jj = np.triu_indices(len(row), 1)
            need.append(row[ii] * L + row[jj])
    n_need = 0
    if need:
        need = np.concatenate(need)
        n_need = len(need)
        pos = np.minimum(np.searchsorted(ekey, need), max(len(ekey) - 1, 0))
        assert len(ekey) and np.all(ekey[pos] == need), "a witnessed pair is missing from E"
    se = rng.choice(len(edges), size=min(n_edges, len(edges)), replace=False) if len(edges) else []
    for e in np.asarray(se, dtype=np.int64).tolist():
        i, j = edges[e]
        bi = ball_idx[ball_ptr[i]:ball_ptr[i + 1]]
        bj = ball_idx[ball_ptr[j]:ball_ptr[j + 1]]
        assert len(np.intersect1d(bi, bj, assume_unique=True)) > 0, f"edge {i}-{j} unwitnessed"
    rep["edge_pairs_checked"] = int(n_need)
    rep["edges_witnessed"] = int(len(se))
    return rep
