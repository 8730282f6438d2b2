"""Python loader for the plain-C oracle (`oracle/bm_oracle.c`).

TEST INFRASTRUCTURE ONLY — only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
module.  It shares no code with the CUDA product path
(``paper_2601_01405_b200``); it only consumes the same seeded inputs from
``workloads/``.

See the header of ``bm_oracle.c`` for what each function computes and the
PAPER.md passages it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "bm_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

DTYPE_CODE = {"f32": 0, "i8": 1, "u8": 2}
METRIC_CODE = {"l2": 0, "l1": 1, "cos": 2}
NP_TO_DTYPE = {np.dtype(np.float32): "f32", np.dtype(np.int8): "i8", np.dtype(np.uint8): "u8"}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2, OpenMP, no fast-math, no FP contraction."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", LIB + ".tmp", SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


class _Cover(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int64), ("landmarks", ctypes.POINTER(ctypes.c_int64)),
                ("M", ctypes.c_int64), ("ball_ptr", ctypes.POINTER(ctypes.c_int64)),
                ("ball_idx", ctypes.POINTER(ctypes.c_int64)),
                ("pt_ptr", ctypes.POINTER(ctypes.c_int64)),
                ("pt_lm", ctypes.POINTER(ctypes.c_int64)),
                ("E", ctypes.c_int64), ("edges", ctypes.POINTER(ctypes.c_int64)),
                ("pairs_evaluated", ctypes.c_int64)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_cover.argtypes = [vp, i32, i64, i32, i32, dbl, vp, vp, vp, i64,
                                     ctypes.POINTER(_Cover)]
        lib.oracle_cover.restype = i32
        lib.oracle_free.argtypes = [ctypes.POINTER(_Cover)]
        lib.oracle_range_query.argtypes = [vp, i32, i64, i32, i32, dbl, i64, vp]
        lib.oracle_range_query.restype = i32
        lib.oracle_pair_distances.argtypes = [vp, i32, i32, i32, vp, vp, i64, vp]
        lib.oracle_pair_inball.argtypes = [vp, i32, i32, i32, dbl, vp, vp, i64, vp]
        lib.oracle_distance.argtypes = [vp, i32, i32, i32, i64, i64]
        lib.oracle_distance.restype = dbl
        lib.oracle_cover_given.argtypes = [vp, i32, i64, i32, i32, dbl, vp, i64, vp, vp, vp,
                                           i64, ctypes.POINTER(_Cover)]
        lib.oracle_cover_given.restype = i32
        lib.oracle_fps.argtypes = [vp, i32, i64, i32, i32, dbl, i64, vp]
        lib.oracle_fps.restype = i64
        lib.oracle_set_threads.argtypes = [i32]
        lib.oracle_set_threads.restype = i32
        _lib = lib
    return _lib


def set_threads(t: int = 0) -> int:
    """Set the OpenMP thread count (0 = leave as is); returns the count in use."""
    return _load().oracle_set_threads(int(t))


@dataclass
class OracleCover:
    landmarks: np.ndarray            # [L] int64 point indices, ascending
    ball_ptr: np.ndarray             # [L+1] int64
    ball_idx: np.ndarray             # [M] int64 point indices
    pt_ptr: np.ndarray               # [n+1] int64
    pt_lm: np.ndarray                # [M] int64 landmark positions
    edges: np.ndarray                # [E, 2] int64
    pairs_evaluated: int = 0
    overrides: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def L(self):
        return int(self.landmarks.shape[0])

    @property
    def M(self):
        return int(self.ball_idx.shape[0])

    @property
    def E(self):
        return int(self.edges.shape[0])


def _arr(ptr, n):
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    return np.ctypeslib.as_array(ptr, shape=(n,)).copy()


def fps(X: np.ndarray, metric: str, eps: float, start: int = 0) -> np.ndarray:
    """Farthest point sampling eps-net (readings F1-F2 in
    bm_oracle.c): the landmark indices in selection order."""
    X = np.ascontiguousarray(X)
    dt = NP_TO_DTYPE[X.dtype]
    n, d = X.shape
    seq = np.zeros(n, dtype=np.int64)
    L = _load().oracle_fps(X.ctypes.data, DTYPE_CODE[dt], n, d, METRIC_CODE[metric], float(eps),
                           int(start), seq.ctypes.data)
    if L < 0:
        raise ValueError("oracle_fps: invalid input")
    return seq[:L].copy()


def cover(X: np.ndarray, metric: str, eps: float, overrides=None, landmarks=None) -> OracleCover:
    """Greedy eps-net + ball membership + 1-skeleton (see bm_oracle.c header).

    overrides: optional iterable of (p, q, bool) — point p, landmark point q.
    landmarks: optional ascending landmark list (e.g. sorted FPS landmarks)
    whose cover is built instead of the greedy's."""
    X = np.ascontiguousarray(X)
    if X.ndim != 2:
        raise ValueError("X must be 2-D")
    dt = NP_TO_DTYPE.get(X.dtype)
    if dt is None:
        raise ValueError(f"unsupported dtype {X.dtype}")
    n, d = X.shape
    lib = _load()
    ov = list(overrides or [])
    if ov:
        op = np.array([o[0] for o in ov], dtype=np.int64)
        oq = np.array([o[1] for o in ov], dtype=np.int64)
        oval = np.array([1 if o[2] else 0 for o in ov], dtype=np.int8)
        args = (op.ctypes.data, oq.ctypes.data, oval.ctypes.data, len(ov))
    else:
        args = (None, None, None, 0)
    c = _Cover()
    if landmarks is not None:
        g = np.ascontiguousarray(np.asarray(landmarks, dtype=np.int64))
        rc = lib.oracle_cover_given(X.ctypes.data if n else None, DTYPE_CODE[dt], n, d,
                                    METRIC_CODE[metric], float(eps), g.ctypes.data, len(g),
                                    *args, ctypes.byref(c))
    else:
        rc = lib.oracle_cover(X.ctypes.data if n else None, DTYPE_CODE[dt], n, d,
                              METRIC_CODE[metric], float(eps), *args, ctypes.byref(c))
    if rc == 1:
        raise ValueError("oracle_cover: invalid input")
    if rc != 0:
        raise MemoryError("oracle_cover: allocation failure")
    try:
        res = OracleCover(
            landmarks=_arr(c.landmarks, c.L), ball_ptr=_arr(c.ball_ptr, c.L + 1),
            ball_idx=_arr(c.ball_idx, c.M), pt_ptr=_arr(c.pt_ptr, n + 1),
            pt_lm=_arr(c.pt_lm, c.M), edges=_arr(c.edges, 2 * c.E).reshape(-1, 2),
            pairs_evaluated=int(c.pairs_evaluated), overrides=len(ov))
    finally:
        lib.oracle_free(ctypes.byref(c))
    return res


def range_query(X: np.ndarray, metric: str, eps: float, q: int) -> np.ndarray:
    """Indices {p : d(x_p, x_q) < eps}, ascending."""
    X = np.ascontiguousarray(X)
    n, d = X.shape
    out = np.zeros(n, dtype=np.uint8)
    rc = _load().oracle_range_query(X.ctypes.data, DTYPE_CODE[NP_TO_DTYPE[X.dtype]], n, d,
                                    METRIC_CODE[metric], float(eps), int(q), out.ctypes.data)
    if rc:
        raise ValueError("oracle_range_query: invalid input")
    return np.nonzero(out)[0].astype(np.int64)


def pair_distances(X: np.ndarray, metric: str, p, q) -> np.ndarray:
    """fp64 distances (Euclidean distance for L2, not squared) for pairs (p[k], q[k])."""
    X = np.ascontiguousarray(X)
    p = np.ascontiguousarray(p, dtype=np.int64)
    q = np.ascontiguousarray(q, dtype=np.int64)
    out = np.empty(p.shape[0], dtype=np.float64)
    _load().oracle_pair_distances(X.ctypes.data, DTYPE_CODE[NP_TO_DTYPE[X.dtype]], X.shape[1],
                                  METRIC_CODE[metric], p.ctypes.data, q.ctypes.data,
                                  p.shape[0], out.ctypes.data)
    return out


def pair_inball(X: np.ndarray, metric: str, eps: float, p, q) -> np.ndarray:
    """The oracle's own in-ball predicate for pairs (p[k], q[k]) -> bool array."""
    X = np.ascontiguousarray(X)
    p = np.ascontiguousarray(p, dtype=np.int64)
    q = np.ascontiguousarray(q, dtype=np.int64)
    out = np.empty(p.shape[0], dtype=np.uint8)
    _load().oracle_pair_inball(X.ctypes.data, DTYPE_CODE[NP_TO_DTYPE[X.dtype]], X.shape[1],
                               METRIC_CODE[metric], float(eps), p.ctypes.data, q.ctypes.data,
                               p.shape[0], out.ctypes.data)
    return out.astype(bool)


def distance(X: np.ndarray, metric: str, p: int, q: int) -> float:
    """Raw oracle distance value (SQUARED for L2) between rows p and q."""
    X = np.ascontiguousarray(X)
    return _load().oracle_distance(X.ctypes.data, DTYPE_CODE[NP_TO_DTYPE[X.dtype]], X.shape[1],
                                   METRIC_CODE[metric], int(p), int(q))


def near_tie_band(X: np.ndarray, metric: str, eps: float, p, q, rel: float = 1e-6) -> np.ndarray:
    """True where |d_fp64(p,q) - eps| <= rel*eps (BASELINE.json north_star tolerance)."""
    dist = pair_distances(X, metric, p, q)
    return np.abs(dist - eps) <= rel * eps
