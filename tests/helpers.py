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
