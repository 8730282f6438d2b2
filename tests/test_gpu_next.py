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


# ---------------------------------------------------------------- FPS (NEXT-2)
def _fps_case(bm, X_, metric, eps, start=0, **kw):
    want = np.sort(O.fps(X_, metric, eps, start))
    cov = bm.cover_build(torch.from_numpy(np.ascontiguousarray(X_)).cuda(), metric, eps,
                         select="fps", fps_start=start, **kw)
    got = cov.numpy()["landmarks"]
    assert np.array_equal(np.asarray(got, dtype=np.int64), want), "FPS landmark set differs"
    return compare(X_, metric, eps, cov, float_path=X_.dtype == np.float32, landmarks=want)


@pytest.mark.parametrize("metric,eps", [("l2", 0.5), ("l1", 0.9), ("cos", 0.05)])
@pytest.mark.parametrize("seed", range(3))
def test_fps_parity_random(bm, metric, eps, seed):
    rng = np.random.default_rng([seed, 21])
    X_ = rng.normal(size=(3000 + 77 * seed, 3)).astype(np.float32)
    _fps_case(bm, X_, metric, eps, start=seed * 11)


@pytest.mark.parametrize("dtype,metric,eps", [("i8", "l2", 6.5), ("u8", "l1", 9.0),
                                              ("i8", "l1", 7.0), ("u8", "l2", 12.0)])
def test_fps_parity_int(bm, dtype, metric, eps):
    rng = np.random.default_rng(5)
    X_ = (rng.integers(-40, 40, size=(4000, 4)).astype(np.int8) if dtype == "i8"
          else rng.integers(0, 90, size=(4000, 4)).astype(np.uint8))
    _fps_case(bm, X_, metric, eps)


@pytest.mark.parametrize("name,m", [("c1", None), ("c2", 20000)])
def test_fps_parity_workloads(bm, name, m):
    w = gen.get(name)
    X_ = gen.generate(w, m)
    _fps_case(bm, X_, w.metric, w.eps)


@pytest.mark.parametrize("path", ["cuda_core", "tensor"])
def test_fps_paths_and_ties(bm, path):
    """Both membership paths; exact-distance ties in the argmax (integer
    lattice: many points at the same max-min distance, lowest index wins) and
    a point at exactly eps (reading F1: it becomes a landmark)."""
    g = np.stack(np.meshgrid(np.arange(12), np.arange(12), np.arange(12)), -1).reshape(-1, 3)
    X_ = (g * 2).astype(np.float32)
    _fps_case(bm, X_, "l2", 4.0, path=path)          # distance exactly eps occurs everywhere
    _fps_case(bm, X_, "l2", 4.0, start=5, path=path)


def test_fps_degenerate(bm):
    one = np.zeros((1, 3), np.float32)
    assert _fps_case(bm, one, "l2", 1.0)["L"] == 1
    same = np.ones((500, 2), np.float32)                 # all distances 0: one landmark
    assert _fps_case(bm, same, "l1", 0.1)["L"] == 1
    far = np.arange(40, dtype=np.float32).reshape(-1, 1) * 10   # all singletons
    assert _fps_case(bm, far, "l2", 1.0)["L"] == 40
    with pytest.raises(Exception):
        bm.cover_build(torch.from_numpy(far).cuda(), "l2", 1.0, select="fps", fps_start=40)


@pytest.mark.parametrize("metric,eps", [("l2", 0.35), ("l1", 0.6)])
def test_fps_pruned_equals_unpruned(bm, metric, eps):
    """FPS with the spatial order and per-warp bounding balls (fps.cu) against
    the unpruned kernel and the oracle, on clustered data where most warps skip."""
    from paper_2601_01405_b200 import bm as B
    rng = np.random.default_rng(31)
    centres = rng.normal(size=(20, 6)) * 8.0
    X_ = (centres[rng.integers(0, 20, size=12000)] + rng.normal(size=(12000, 6)) * 0.3).astype(np.float32)
    t = torch.from_numpy(X_).cuda()
    a = bm.cover_build(t, metric, eps, select="fps")
    b = bm.cover_build(t, metric, eps, select="fps", flags=B.FLAG_NO_PRUNE)
    na, nb = a.numpy(), b.numpy()
    for k in na:
        assert np.array_equal(na[k], nb[k]), k
    want = np.sort(O.fps(X_, metric, eps))
    assert np.array_equal(np.asarray(na["landmarks"], dtype=np.int64), want)
