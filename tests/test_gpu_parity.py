"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Marked `gpu`; run on a B200.  Sizes span several greedy tiles (T down to 32)
and ragged tails.  Full C1 and C2 are compared array by array here; full C4
and the full-size C3 / C5 validity checks (LFMIS certificate, CSR transpose,
>= 1e7 sampled pairs re-decided by the oracle, complete rows / columns,
sampled edges) and the near-tie completeness tests are in
test_gpu_fullsize.py.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from tests.helpers import balls_of, case_arrays, lfmis_certificate  # noqa: E402
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


def run(bm, X, metric, eps, **kw):
    t = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    return bm.cover_build(t, metric, eps, **kw)


def test_golden_cases_on_gpu(bm, golden_cases):
    for case in golden_cases:
        X, eps = case_arrays(case)
        cov = run(bm, X, case["metric"], eps)
        a = cov.numpy()
        assert a["landmarks"].tolist() == case["landmarks"], case["name"]
        assert balls_of(a["ball_ptr"], a["ball_idx"]) == case["balls"], case["name"]
        assert a["edges"].tolist() == case["edges"], case["name"]


@pytest.mark.parametrize("metric,dtype", [("l2", "f32"), ("l1", "f32"), ("cos", "f32"),
                                          ("l2", "i8"), ("l2", "u8"), ("l1", "i8"),
                                          ("l1", "u8")])
@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("tile", [32, 1024])
def test_random_clouds(bm, metric, dtype, seed, tile):
    rng = np.random.default_rng([seed, 11])
    n = int(rng.integers(500, 3000))
    d = int(rng.integers(1, 20))
    if dtype == "f32":
        X = gen.random_cloud(n, d, "f32", seed=seed)
        eps = {"l2": 0.3 * math.sqrt(d), "l1": 0.25 * d, "cos": 0.08}[metric]
    else:
        X = gen.random_cloud(n, d, dtype, seed=seed, lo=-20 if dtype == "i8" else 0, hi=20)
        eps = {"l2": math.sqrt(30.0 * d + 0.5), "l1": 8.0 * d + 0.5}[metric]
    cov = run(bm, X, metric, eps, tile=tile)
    compare(X, metric, eps, cov, float_path=dtype == "f32")


@pytest.mark.parametrize("d", [3, 10, 16, 33, 64, 100, 257])
def test_dimension_widths(bm, d):
    """Register-row widths and the wide variant (d > 64 floats / 256 bytes)."""
    n = 1500
    X = gen.random_cloud(n, d, "f32", seed=d)
    eps = 0.33 * math.sqrt(d)
    compare(X, "l2", eps, run(bm, X, "l2", eps, tile=64), float_path=True)
    Xi = gen.random_cloud(n, d, "u8", seed=d, lo=0, hi=255)
    epsi = math.sqrt(d * 4000.0 + 0.5)
    compare(Xi, "l2", epsi, run(bm, Xi, "l2", epsi, tile=64), float_path=False)


def test_c1_full_bit_exact(bm):
    w = gen.get("c1")
    X = gen.generate(w)
    r = compare(X, w.metric, w.eps, run(bm, X, w.metric, w.eps), float_path=False)
    assert r["L"] > 1 and r["E"] > 0


@pytest.mark.parametrize("tile", [32, 256, 1024])
def test_c2_full_tile_invariance(bm, tile):
    w = gen.get("c2")
    X = gen.generate(w)
    o = O.cover(X, w.metric, w.eps)
    cov = run(bm, X, w.metric, w.eps, tile=tile)
    compare(X, w.metric, w.eps, cov, float_path=True, oracle_result=o, tie_rate_limit=True)


def test_c4_prefix_bit_exact(bm):
    w = gen.get("c4")
    X = gen.generate(w, 6000)
    compare(X, w.metric, w.eps, run(bm, X, w.metric, w.eps), float_path=False)


@pytest.mark.parametrize("name,m", [("c3_e8", 20000), ("c3_e4", 8000), ("c5_l1", 60000),
                                    ("c5_cos", 60000)])
def test_prefix_parity(bm, name, m):
    w = gen.get(name)
    X = gen.generate(w, m)
    compare(X, w.metric, w.eps, run(bm, X, w.metric, w.eps), float_path=True,
            tie_rate_limit=True)


def test_edge_cases(bm):
    # n = 1
    X = np.array([[1.5, -2.0]], dtype=np.float32)
    a = run(bm, X, "l2", 1.0).numpy()
    assert a["landmarks"].tolist() == [0] and a["ball_idx"].tolist() == [0]
    assert a["edges"].shape == (0, 2)
    # d = 1, all duplicates
    X = np.zeros((5000, 1), dtype=np.float32)
    a = run(bm, X, "l2", 0.5).numpy()
    assert a["landmarks"].tolist() == [0] and a["ball_idx"].tolist() == list(range(5000))
    # eps smaller than every distance -> all landmarks, singleton balls, no edges
    X = np.arange(3000, dtype=np.float32).reshape(-1, 1)
    a = run(bm, X, "l2", 0.5, tile=128).numpy()
    assert a["landmarks"].tolist() == list(range(3000))
    assert a["ball_idx"].tolist() == list(range(3000)) and a["edges"].shape[0] == 0
    # ragged n around the tile size
    for n in (31, 32, 33, 1023, 1025):
        X = gen.random_cloud(n, 4, "f32", seed=n)
        compare(X, "l2", 0.4, run(bm, X, "l2", 0.4, tile=32), float_path=True)


def test_host_path_equals_device_path(bm):
    w = gen.get("c2")
    X = gen.generate(w, 30000)
    a = run(bm, X, w.metric, w.eps).numpy()
    h = bm.cover_build_host(X, w.metric, w.eps).numpy()
    for k in a:
        assert np.array_equal(a[k], h[k]), k


def test_determinism(bm):
    w = gen.get("c2")
    X = gen.generate(w, 50000)
    a = run(bm, X, w.metric, w.eps, tile=256).numpy()
    b = run(bm, X, w.metric, w.eps, tile=256).numpy()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_error_codes(bm):
    from paper_2601_01405_b200 import bm as B
    t = torch.zeros((4, 2), dtype=torch.float32, device="cuda")
    p = t.data_ptr()
    assert B.raw_build(0, "f32", 4, 2, "l2", 1.0)[0] == B.BM_EINVAL
    assert B.raw_build(p, "f32", 0, 2, "l2", 1.0)[0] == B.BM_EINVAL
    assert B.raw_build(p, "f32", 4, 0, "l2", 1.0)[0] == B.BM_EINVAL
    for e in (0.0, -1.0, float("nan"), float("inf")):
        assert B.raw_build(p, "f32", 4, 2, "l2", e)[0] == B.BM_EINVAL
    ti = torch.zeros((4, 2), dtype=torch.int8, device="cuda")
    assert B.raw_build(ti.data_ptr(), "i8", 4, 2, "cos", 1.0)[0] == B.BM_EUNSUPPORTED
    assert B.raw_build(p, 7, 4, 2, "l2", 1.0)[0] == B.BM_EUNSUPPORTED
    assert B.raw_build(p, "f32", 4, 2, 9, 1.0)[0] == B.BM_EUNSUPPORTED
    assert B.raw_build(p, "f32", 2**31, 2, "l2", 1.0)[0] == B.BM_EOVERFLOW
    t[1, 0] = float("nan")
    rc, _ = B.raw_build(t.data_ptr(), "f32", 4, 2, "l2", 1.0)
    assert rc == B.BM_EINVAL
    assert "non-finite" in B.load().bm_last_error().decode()
    B.load().bm_free(None)  # NULL-safe


def test_no_leak(bm):
    w = gen.get("c1")
    X = torch.from_numpy(gen.generate(w)).cuda()
    for _ in range(3):
        bm.cover_build(X, w.metric, w.eps).free()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(50):
        bm.cover_build(X, w.metric, w.eps).free()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 64 << 20


def test_radix_sort_matches_torch(bm):
    from paper_2601_01405_b200 import bm as B
    g = torch.Generator().manual_seed(0)
    for n, bits in [(1, 8), (1000, 12), (100_003, 40), (2_000_000, 27)]:
        k = torch.randint(0, 2 ** bits, (n,), generator=g, dtype=torch.int64)
        d = k.cuda()
        B.radix_sort_u64(d, bits)
        assert torch.equal(d.cpu(), torch.sort(k).values)


def test_scan_matches_cumsum(bm):
    from paper_2601_01405_b200 import bm as B
    for n in (1, 4095, 4096, 4097, 1_000_001):
        x = torch.randint(0, 100, (n,), dtype=torch.int64).cuda()
        out, tot = B.exclusive_scan_i64(x)
        ref = torch.cumsum(x, 0) - x
        assert torch.equal(out, ref) and tot == int(x.sum())


def test_resolve_matches_cpu_lfmis(bm):
    from paper_2601_01405_b200 import bm as B
    rng = np.random.default_rng(5)
    for nc in (1, 31, 32, 33, 500, 1024):
        for dens in (0.0, 0.01, 0.2, 0.9):
            A = np.tril(rng.random((nc, nc)) < dens, -1)
            words = np.zeros((nc, (nc + 31) // 32), dtype=np.uint32)
            for a in range(nc):
                for b in np.nonzero(A[a])[0]:
                    words[a, b // 32] |= np.uint32(1 << (b % 32))
            got = B.resolve_tile(words, nc)
            sel = []
            for a in range(nc):
                if not any(A[a, b] for b in sel):
                    sel.append(a)
            ref = np.zeros(nc, dtype=np.uint8)
            ref[sel] = 1
            assert np.array_equal(got, ref), (nc, dens)


def test_full_c2_certificate(bm):
    w = gen.get("c2")
    X = gen.generate(w)
    a = run(bm, X, w.metric, w.eps).numpy()
    assert lfmis_certificate(a["landmarks"], a["pt_ptr"], a["pt_lm"], len(X)) == []


def test_capacity_fallbacks(bm):
    """An undersized key buffer takes the documented recovery path (one
    exact-capacity membership recount) and gives the same answer, on both
    contraction paths."""
    w = gen.get("c2")
    X = gen.generate(w, 20000)
    t = torch.from_numpy(X).cuda()
    ref = run(bm, X, w.metric, w.eps).numpy()
    small = bm.cover_build(t, w.metric, w.eps, key_cap=1000).numpy()
    for k in ref:
        assert np.array_equal(ref[k], small[k]), k
    w3 = gen.get("c3_e8")
    X3 = gen.generate(w3, 6000)
    t3 = torch.from_numpy(X3).cuda()
    cov = bm.cover_build(t3, w3.metric, w3.eps, path="tensor", key_cap=100)
    assert cov.stats.path_used == 2
    compare(X3, w3.metric, w3.eps, cov, float_path=True)


@pytest.mark.parametrize("seed", range(3))
def test_l1_prefilter_equivalence(bm, seed):
    """The 8-bit SAD prefilter of the L1 membership pass only skips pairs it
    proves out: results equal the unfiltered fp32 path and the oracle, also
    for wide coordinate ranges (coarse quantisation), exact-eps distances and
    d not a multiple of 4."""
    from paper_2601_01405_b200 import bm as B
    rng = np.random.default_rng([seed, 77])
    n, d = 4000, [16, 7, 33][seed]
    X = rng.random((n, d)).astype(np.float32)
    if seed == 1:
        X[::50] *= 1000.0            # a few far outliers: coarse 8-bit scale
    if seed == 2:
        X[1::2] = X[0::2][: n // 2]  # duplicates, then shift coordinate 0 by exactly eps
        X[1::2, 0] += np.float32(0.5)
    eps = 0.5 if seed == 2 else 0.25 * d / 4
    t = torch.from_numpy(X).cuda()
    a = bm.cover_build(t, "l1", eps, tile=256)
    b = bm.cover_build(t, "l1", eps, tile=256, flags=B.FLAG_NO_L1_PREFILTER)
    na, nb = a.numpy(), b.numpy()
    for k in na:
        assert np.array_equal(na[k], nb[k]), k
    compare(X, "l1", eps, a, float_path=True)


@pytest.mark.parametrize("metric,eps", [("l2", 0.006), ("l1", 0.008), ("cos", 4e-5)])
def test_edges_large_L_paths(bm, metric, eps):
    """L > 4096: the default row-union emission (per-row-item dedup, sort,
    unique), the per-point pair emission and the strictly-upper bit triangle
    (edges.cu) agree with each other and with the oracle."""
    from paper_2601_01405_b200 import bm as B
    rng = np.random.default_rng(17)
    X = rng.random((12000, 3 if metric == "cos" else 2)).astype(np.float32)
    t = torch.from_numpy(X).cuda()
    a = bm.cover_build(t, metric, eps, flags=B.FLAG_EDGE_ROWS)
    b = bm.cover_build(t, metric, eps, flags=B.FLAG_EDGE_POINT_PAIRS)
    c = bm.cover_build(t, metric, eps, flags=B.FLAG_EDGE_TRIANGLE)
    assert a.L > 4096 and a.E > 100, (a.L, a.E)
    na, nb, nc = a.numpy(), b.numpy(), c.numpy()
    for k in na:
        assert np.array_equal(na[k], nb[k]), k
        assert np.array_equal(na[k], nc[k]), k
    assert a.P == b.P == c.P
    compare(X, metric, eps, a, float_path=True)


def test_edges_row_union_heavy_rows(bm):
    """Row items: a ball of 3000 points (six items of 512 members) whose
    points all lie in several other balls, plus a sparse remainder — every
    (i, j) a heavy row repeats across its items must still come out once."""
    rng = np.random.default_rng(23)
    blob = (0.5 + 0.01 * rng.standard_normal((3000, 2))).astype(np.float32)
    rest = rng.random((9000, 2)).astype(np.float32)
    X = np.concatenate([blob, rest])[rng.permutation(12000)]
    t = torch.from_numpy(X).cuda()
    from paper_2601_01405_b200 import bm as B
    a = bm.cover_build(t, "l2", 0.0075, flags=B.FLAG_EDGE_ROWS)
    assert a.L > 4096, a.L
    compare(X, "l2", 0.0075, a, float_path=True)


@pytest.mark.parametrize("tile", [2048, 8192])
@pytest.mark.parametrize("dense", [False, True])
def test_big_tile_invariance(bm, tile, dense):
    """Tiles of more than 1024 candidates (k_resolve_big): the sparse-list
    rounds and the dense sub-tile path both give the oracle's cover (A11)."""
    from paper_2601_01405_b200 import bm as B
    w = gen.get("c2")
    X = gen.generate(w)
    cov = run(bm, X, w.metric, w.eps, tile=tile, flags=B.FLAG_DENSE_RESOLVE if dense else 0)
    assert cov.stats.tile_used == tile
    compare(X, w.metric, w.eps, cov, float_path=True, tie_rate_limit=True)


@pytest.mark.parametrize("path", ["cuda_core", "tensor"])
def test_big_tile_chains(bm, path):
    """A long in-tile dependency chain (collinear points at unit spacing, eps
    1.5: candidate i is adjacent only to i - 1) exceeds the sparse rounds'
    budget and must fall back to the in-order dense path; a dense clump
    overflows the non-zero word list."""
    X = np.arange(20000, dtype=np.float32).reshape(-1, 1)
    a = run(bm, X, "l2", 1.5, tile=8192, path=path).numpy()
    assert a["landmarks"].tolist() == list(range(0, 20000, 2))
    rng = np.random.default_rng(9)
    Y = (rng.random((12000, 3)) * 0.2).astype(np.float32)
    Y[6000:] += 5.0 * rng.random((6000, 3)).astype(np.float32)
    compare(Y, "l2", 0.05, run(bm, Y, "l2", 0.05, tile=8192, path=path), float_path=True)


@pytest.mark.parametrize("name,m", [("c3_e8", 30000), ("c3_e4", 20000)])
def test_big_tile_pruned(bm, name, m):
    """The pruned contraction with 8192-column tiles (multi-word live-chunk
    bitmaps, streamed landmark tiles) against the 1024 tiles and the oracle."""
    from paper_2601_01405_b200 import bm as B
    w = gen.get(name)
    X = gen.generate(w, m)
    t = torch.from_numpy(X).cuda()
    big = bm.cover_build(t, w.metric, w.eps, path="tensor", tile=8192, flags=B.FLAG_FORCE_PRUNE)
    small = bm.cover_build(t, w.metric, w.eps, path="tensor", tile=1024,
                           flags=B.FLAG_FORCE_PRUNE)
    nb, ns = big.numpy(), small.numpy()
    for k in nb:
        assert np.array_equal(nb[k], ns[k]), k
    assert big.stats.tc_tiles_skipped > 0
    compare(X, w.metric, w.eps, big, float_path=True)
