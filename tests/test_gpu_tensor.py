"""tcgen05 membership contraction (tc.cu): raw accumulator checks and
tensor-path parity against the oracle."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from tests.parity import compare  # noqa: E402
from workloads import gen  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_01405_b200 as pkg
    pkg.load()
    return pkg


def tf32_rna(x: np.ndarray) -> np.ndarray:
    """Round fp32 to tf32, nearest with ties away from zero (cvt.rna.tf32.f32)."""
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    b = ((b + 0x1000) & ~np.uint64(0x1FFF)) & np.uint64(0xFFFFFFFF)
    return b.astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("n,d,L", [(300, 3, 70), (1000, 17, 333), (1500, 64, 700),
                                   (700, 100, 257), (129, 128, 65),
                                   # wide rows: A atoms streamed with the B atoms (ABUF = 0)
                                   (300, 129, 70), (600, 200, 300), (600, 500, 513),
                                   (400, 1000, 129), (130, 1024, 33)])
def test_tc_gram_tf32(bm, n, d, L):
    from paper_2601_01405_b200 import bm as B
    rng = np.random.default_rng(n + d)
    X = rng.normal(size=(n, d)).astype(np.float32) * 3
    lm = np.sort(rng.choice(n, size=L, replace=False)).astype(np.int32)
    got = B.tc_gram(torch.from_numpy(X).cuda(), torch.from_numpy(lm).cuda()).cpu().numpy()
    Xr = tf32_rna(X).astype(np.float64)
    exp = Xr @ Xr[lm].T
    K = 8 * math.ceil(d * 4 / 32)
    bound = 4 * K * 2.0 ** -23 * (np.abs(Xr) @ np.abs(Xr[lm]).T) + 1e-30
    err = np.abs(got.astype(np.float64) - exp)
    assert np.all(err <= bound), float((err / bound).max())


@pytest.mark.parametrize("dtype", ["u8", "i8"])
@pytest.mark.parametrize("n,d,L", [(300, 3, 70), (1000, 32, 257), (777, 100, 300),
                                   (600, 784, 513), (513, 896, 77), (300, 1000, 100),
                                   (200, 4096, 50)])
def test_tc_gram_int8_exact(bm, dtype, n, d, L):
    from paper_2601_01405_b200 import bm as B
    rng = np.random.default_rng(n * 7 + d)
    if dtype == "u8":
        X = rng.integers(0, 256, size=(n, d)).astype(np.uint8)
    else:
        X = rng.integers(-128, 128, size=(n, d)).astype(np.int8)
    lm = np.sort(rng.choice(n, size=L, replace=False)).astype(np.int32)
    got = B.tc_gram(torch.from_numpy(X).cuda(), torch.from_numpy(lm).cuda()).cpu().numpy()
    Xi = X.astype(np.int64)
    assert np.array_equal(got.astype(np.int64), Xi @ Xi[lm].T)


@pytest.mark.parametrize("name,m", [("c3_e8", 20000), ("c3_e4", 12000), ("c3_e2", 6000),
                                    ("c4", 8000)])
def test_tensor_path_parity(bm, name, m):
    w = gen.get(name)
    X = gen.generate(w, m)
    cov = bm.cover_build(torch.from_numpy(X).cuda(), w.metric, w.eps, path="tensor")
    assert cov.stats.path_used == 2
    compare(X, w.metric, w.eps, cov, float_path=w.dtype == "f32", tie_rate_limit=True)


@pytest.mark.parametrize("d", [32, 33, 64, 100, 128, 200, 513, 1000])
@pytest.mark.parametrize("dtype", ["f32", "u8", "i8"])
def test_tensor_path_random(bm, d, dtype):
    n = 3000
    if dtype == "f32":
        X = gen.random_cloud(n, d, "f32", seed=d)
        eps = 0.36 * math.sqrt(d)
    else:
        X = gen.random_cloud(n, d, dtype, seed=d, lo=-60 if dtype == "i8" else 0, hi=60)
        eps = math.sqrt(d * 1100.0 + 0.5)
    cov = bm.cover_build(torch.from_numpy(X).cuda(), "l2", eps, path="tensor", tile=256)
    compare(X, "l2", eps, cov, float_path=dtype == "f32")
    # near-boundary adversarial: exact duplicates shifted by tiny offsets
    if dtype == "f32":
        Y = X.copy()
        Y[1::2] = Y[0::2][: len(Y[1::2])] + np.float32(eps / math.sqrt(d)) * (1 + 1e-6)
        cov = bm.cover_build(torch.from_numpy(Y).cuda(), "l2", eps, path="tensor")
        compare(Y, "l2", eps, cov, float_path=True)


@pytest.mark.parametrize("d", [3, 16, 64, 100, 300])
def test_tensor_path_cosine(bm, d):
    """Cosine distance on tcgen05 (Gram of the normalised rows, rigorous band,
    fp64 recheck with the zero-vector rule): equal to the oracle, with zero
    rows, duplicate directions and points exactly at eps."""
    rng = np.random.default_rng(d)
    n = 3000
    X = rng.normal(size=(n, d)).astype(np.float32)
    X[::97] = 0.0                                  # zero vectors (reading A7)
    X[1::5] = X[0::5][: len(X[1::5])] * np.float32(3.0)   # same direction: distance 0
    eps = 0.05 if d > 3 else 0.02
    cov = bm.cover_build(torch.from_numpy(X).cuda(), "cos", eps, path="tensor", tile=256)
    assert cov.stats.path_used == 2
    compare(X, "cos", eps, cov, float_path=True)


def test_tensor_path_cosine_c5_prefix(bm):
    w = gen.get("c5_cos")
    X = gen.generate(w, 60000)
    cov = bm.cover_build(torch.from_numpy(X).cuda(), w.metric, w.eps, path="tensor")
    assert cov.stats.path_used == 2
    compare(X, w.metric, w.eps, cov, float_path=True, tie_rate_limit=True)


@pytest.mark.parametrize("d", [1, 2, 3, 7, 8, 11, 16])
def test_tensor_path_l1(bm, d):
    """L1 on tcgen05 (thermometer-code Gram): the signed int8
    contraction only proves pairs out; results equal the CUDA-core path and
    the oracle for widths with one and two K atoms, also with exact-eps
    shifts along one axis and a few far outliers (coarse levels)."""
    rng = np.random.default_rng([d, 0x11])
    n = 3000
    X = rng.random((n, d)).astype(np.float32)
    eps = 0.3 * d ** 0.75
    X[1::7] = X[0::7][: len(X[1::7])]
    X[1::7, 0] += np.float32(eps)                 # |dx| = eps exactly along axis 0
    t = torch.from_numpy(X).cuda()
    a = bm.cover_build(t, "l1", eps, path="tensor", tile=256)
    b = bm.cover_build(t, "l1", eps, path="cuda_core", tile=256)
    assert a.stats.path_used == 2 and b.stats.path_used == 1
    na, nb = a.numpy(), b.numpy()
    for k in na:
        assert np.array_equal(na[k], nb[k]), k
    compare(X, "l1", eps, a, float_path=True)
    Y = X.copy()
    Y[::61] *= 50.0                               # outliers widen the level spacing
    a = bm.cover_build(torch.from_numpy(Y).cuda(), "l1", eps, path="tensor")
    compare(Y, "l1", eps, a, float_path=True)


def test_tensor_path_l1_unsupported_width(bm):
    from paper_2601_01405_b200 import bm as B
    X = torch.rand(100, 17, device="cuda")
    with pytest.raises(B.BMError):
        bm.cover_build(X, "l1", 1.0, path="tensor")


def test_tensor_path_l1_c5_prefix(bm):
    w = gen.get("c5_l1")
    X = gen.generate(w, 60000)
    cov = bm.cover_build(torch.from_numpy(X).cuda(), w.metric, w.eps, path="tensor")
    assert cov.stats.path_used == 2
    compare(X, w.metric, w.eps, cov, float_path=True, tie_rate_limit=True)


@pytest.mark.parametrize("name,m", [("c3_e8", 20000), ("c3_e4", 12000), ("c3_e2", 6000),
                                    ("c2", None)])
def test_pruned_contraction_parity(bm, name, m):
    """Tile-level pruning (cells.cu): forced on below its size threshold, the
    cover equals the unpruned one and the oracle's."""
    from paper_2601_01405_b200 import bm as B
    w = gen.get(name)
    X = gen.generate(w, m)
    t = torch.from_numpy(X).cuda()
    a = bm.cover_build(t, w.metric, w.eps, path="tensor", flags=B.FLAG_FORCE_PRUNE)
    b = bm.cover_build(t, w.metric, w.eps, path="tensor", flags=B.FLAG_NO_PRUNE)
    na, nb = a.numpy(), b.numpy()
    for k in na:
        assert np.array_equal(na[k], nb[k]), k
    compare(X, w.metric, w.eps, a, float_path=True)


@pytest.mark.parametrize("seed", range(3))
def test_pruned_contraction_clusters(bm, seed):
    """Well-separated clusters (most tiles pruned), points at exactly eps and
    just inside / outside it across cluster borders."""
    from paper_2601_01405_b200 import bm as B
    rng = np.random.default_rng([seed, 77])
    d, k = 24, 12
    centres = rng.normal(size=(k, d)) * 20.0
    X = (centres[rng.integers(0, k, size=9000)] + rng.normal(size=(9000, d))).astype(np.float32)
    eps = 3.0
    X[1::97] = X[0::97][: len(X[1::97])] + np.float32(eps / math.sqrt(d))   # |dx| = eps
    t = torch.from_numpy(X).cuda()
    a = bm.cover_build(t, "l2", eps, path="tensor", flags=B.FLAG_FORCE_PRUNE, tile=256)
    b = bm.cover_build(t, "l2", eps, path="tensor", flags=B.FLAG_NO_PRUNE, tile=256)
    na, nb = a.numpy(), b.numpy()
    for key in na:
        assert np.array_equal(na[key], nb[key]), key
    compare(X, "l2", eps, a, float_path=True)
