"""Full-size GPU validity.

At BASELINE.json's full sizes the plain oracle would take hours (C3, C5), so
the CUDA cover of the full workload, in the launch configuration bench.py
times, is checked by properties that hold at any size plus oracle re-decisions
of sampled pairs (tests/helpers.py fullsize_validity): the LFMIS certificate,
the CSR transpose, every reported membership, >= 1e7 uniform pairs, complete
rows / columns and sampled edges.  C1, C2 (test_gpu_parity.py) and C4 (here)
are small enough for the full oracle and are compared array by array.

A report per config is printed and, if BM_VALIDITY_LOG names a file, appended
to it as one JSON line (committed under profiles/).
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from tests.helpers import fullsize_validity  # noqa: E402
from tests.parity import compare  # noqa: E402
from workloads import gen  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def bm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_01405_b200 as pkg
    pkg.load()
    return pkg


def _log(rep):
    print(json.dumps(rep))
    path = os.environ.get("BM_VALIDITY_LOG")
    if path:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "a") as f:
            f.write(json.dumps(rep) + "\n")


@pytest.mark.parametrize("name,path", [("c3_e2", "auto"), ("c3_e4", "auto"), ("c3_e8", "auto"),
                                       ("c5_l1", "auto"), ("c5_l1", "tensor"), ("c5_cos", "auto")])
def test_fullsize_validity(bm, name, path):
    w = gen.get(name)
    X = gen.generate(w)
    cov = bm.cover_build(torch.from_numpy(X).cuda(), w.metric, w.eps, path=path)
    assert cov.stats.n_near_ties == len(cov.near_ties), "near-tie list truncated"
    a = cov.numpy()
    path = ["auto", "cuda_core", "tensor"][cov.stats.path_used]
    nt = cov.near_ties
    cov.free()
    rep = fullsize_validity(X, w.metric, w.eps, a, nt[:, :2] if len(nt) else nt, seed=7)
    rep.update({"workload": name, "path": path, "eps": w.eps, "metric": w.metric})
    _log(rep)
    assert rep["pairs_rechecked"] >= 10_000_000


def test_c4_full_bit_exact(bm):
    """Full C4 (70,000 x 784 uint8, integer Euclidean): every array bit-exact
    against the full oracle (SURVEY §8(c) parity rule for integer workloads)."""
    w = gen.get("c4")
    X = gen.generate(w)
    cov = bm.cover_build(torch.from_numpy(X).cuda(), w.metric, w.eps)
    r = compare(X, w.metric, w.eps, cov, float_path=False)
    r.update({"workload": "c4", "check": "full oracle, bit-exact",
              "path": ["auto", "cuda_core", "tensor"][cov.stats.path_used]})
    _log(r)


def _tie_cloud(kind, seed):
    """Clouds with many pairs at (or within 0.3e-6 eps of) distance exactly eps."""
    rng = np.random.default_rng([seed, 0x71E])
    if kind == "lattice":      # integer lattice, eps = lattice spacing: exact ties
        g = np.stack(np.meshgrid(np.arange(40), np.arange(40), indexing="ij"), -1).reshape(-1, 2)
        X = g[rng.permutation(len(g))].astype(np.float32)
        return X, 1.0
    if kind == "shifted":      # duplicates shifted by eps (1 +- tiny) along a random axis
        base = (rng.random((800, 6)) * 40.0).astype(np.float32)
        sh = base.copy()
        ax = rng.integers(0, 6, 800)
        delta = np.float32(2.0) * (np.float32(1.0) + rng.choice([-3e-7, 0.0, 3e-7], 800).astype(np.float32))
        sh[np.arange(800), ax] += delta
        X = np.concatenate([base, sh])[rng.permutation(1600)]
        return X.astype(np.float32), 2.0
    if kind == "l1_lattice":
        g = np.stack(np.meshgrid(np.arange(30), np.arange(30), np.arange(3), indexing="ij"),
                     -1).reshape(-1, 3)
        return g[rng.permutation(len(g))].astype(np.float32), 2.0
    # cosine: directions at exact angles on a circle, several radii
    k = rng.integers(0, 24, 1500)
    r = rng.integers(1, 5, 1500).astype(np.float64)
    th = k * (np.pi / 12.0)
    X = np.stack([r * np.cos(th), r * np.sin(th)], 1).astype(np.float32)
    return X, 1.0 - float(np.cos(np.pi / 12.0))


@pytest.mark.parametrize("kind,metric", [("lattice", "l2"), ("shifted", "l2"),
                                         ("l1_lattice", "l1"), ("cos", "cos")])
@pytest.mark.parametrize("path", ["auto", "tensor", "cuda_core"])
def test_near_tie_completeness(bm, kind, metric, path):
    """north_star: near-tie pairs "are reported" — the GPU's near-tie list must
    equal the oracle's full set of in-band (point, landmark) pairs of the final
    cover, not merely a subset of the band."""
    X, eps = _tie_cloud(kind, 3)
    t = torch.from_numpy(X).cuda()
    cov = bm.cover_build(t, metric, eps, path=path, tile=256)
    assert cov.stats.n_near_ties == len(cov.near_ties)
    compare(X, metric, eps, cov, float_path=True)     # parity after overrides
    lms = cov.numpy()["landmarks"].astype(np.int64)
    n = len(X)
    p = np.repeat(np.arange(n, dtype=np.int64), len(lms))
    q = np.tile(lms, n)
    band = O.near_tie_band(X, metric, eps, p, q)
    want = set(zip(p[band].tolist(), q[band].tolist()))
    got = set(zip(cov.near_ties[:, 0].tolist(), cov.near_ties[:, 1].tolist()))
    assert len(want) > 0, "the cloud has no near ties"
    assert got == want, (len(got), len(want), sorted(want - got)[:5], sorted(got - want)[:5])
