"""GPU parity of the §8(f) rows built so far — coloring (NEXT-1)
and the k-skeleton (NEXT-3, Def 2.2) — against the oracle of
oracle/extensions.py on the oracle's own (parity-checked) cover."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import extensions as X  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.parity import compare  # noqa: E402
from workloads import gen  # noqa: E402

pytestmark = pytest.mark.gpu

EXACT = ("median", "min", "max", "mode", "range")
ALL = ("mean", "median", "trimmed", "min", "max", "mode", "variance", "range")


@pytest.fixture(scope="module")
def bm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_01405_b200 as pkg
    pkg.load()
    return pkg


def _covers(bm, X_, metric, eps, float_path):
    cov = bm.cover_build(torch.from_numpy(np.ascontiguousarray(X_)).cuda(), metric, eps)
    compare(X_, metric, eps, cov, float_path=float_path)   # identical covers first
    ov = [(int(p), int(q), bool(v)) for p, q, v in cov.near_ties] if float_path else []
    return cov, O.cover(X_, metric, eps, overrides=ov)


@pytest.mark.parametrize("name,m", [("c1", None), ("c2", 20000), ("c5_l1", 20000)])
def test_color_parity(bm, name, m):
    w = gen.get(name)
    X_ = gen.generate(w, m)
    cov, oc = _covers(bm, X_, w.metric, w.eps, w.dtype == "f32")
    rng = np.random.default_rng(3)
    f = X_[:, 0].astype(np.float32) + rng.normal(size=len(X_)).astype(np.float32) * 0.25
    labels = rng.integers(0, 7, size=len(X_)).astype(np.int32)
    for vals in (f, labels):
        t = torch.from_numpy(vals).cuda()
        for agg in ALL:
            got = bm.color(cov, t, agg, 0.2).cpu().numpy()
            want = X.color(oc.ball_ptr, oc.ball_idx, vals, agg, 0.2)
            if agg in EXACT:
                assert np.array_equal(got, want), (agg, vals.dtype)
            else:   # fp64 sums in a different order
                assert np.allclose(got, want, rtol=1e-12, atol=1e-12 * max(1.0, np.abs(want).max())), agg


def test_color_edge_cases(bm):
    """Trimmed alpha bounds, labels with ties, single-point balls."""
    from paper_2601_01405_b200 import bm as B
    X_ = np.arange(50, dtype=np.float32).reshape(-1, 1) * 3   # eps 1: all singleton balls
    cov = bm.cover_build(torch.from_numpy(X_).cuda(), "l2", 1.0)
    v = torch.arange(50, dtype=torch.float32, device="cuda")
    for agg in ALL:
        got = bm.color(cov, v, agg, 0.4).cpu().numpy()
        want = np.zeros(50) if agg in ("variance", "range") else np.arange(50.0)
        assert np.array_equal(got, want), agg
    with pytest.raises(B.BMError):
        bm.color(cov, v, "trimmed", 0.5)


@pytest.mark.parametrize("name,m,ks", [("c1", None, (1, 2, 3)), ("c2", 20000, (1, 2)),
                                       ("c4", 4000, (2,))])
def test_skeleton_parity(bm, name, m, ks):
    w = gen.get(name)
    X_ = gen.generate(w, m)
    cov, oc = _covers(bm, X_, w.metric, w.eps, w.dtype == "f32")
    for k in ks:
        got = bm.skeleton(cov, k).cpu().numpy().astype(np.int64)
        want = X.skeleton(oc.pt_ptr, oc.pt_lm, k)
        assert np.array_equal(got, want), k
        if k == 1:
            assert np.array_equal(got, oc.edges.reshape(-1, 2))


def test_skeleton_overflow_guard(bm):
    from paper_2601_01405_b200 import bm as B
    w = gen.get("c1")
    X_ = gen.generate(w)
    cov = bm.cover_build(torch.from_numpy(X_).cuda(), w.metric, w.eps)
    with pytest.raises(B.BMError):
        bm.skeleton(cov, 2, max_emit=10)
