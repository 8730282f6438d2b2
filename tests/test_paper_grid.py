"""Host logic of the paper-grid measurement (PAPER.md:263,
P:318-356 [§4.3]): the power-law fit against closed forms and a seeded noise
model, the cube generator's contract, and (GPU) parity of grid cells."""
import math
import sys
import os

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from paper_grid import fit_power_law  # noqa: E402

from workloads import gen  # noqa: E402

GRID_D = np.array(gen.PAPER_GRID_D, dtype=np.float64)


def test_fit_exact_square():
    """y = x^2 -> p = 2, k = 1, R^2 = 1 (log-linear exactly)."""
    f = fit_power_law(GRID_D, GRID_D ** 2)
    assert abs(f["p"] - 2.0) < 1e-9 and abs(f["k"] - 1.0) < 1e-9 and abs(f["r2"] - 1.0) < 1e-9


def test_fit_exact_prefactor():
    """y = 3 x^1.5 -> p = 1.5, k = 3."""
    f = fit_power_law(GRID_D, 3.0 * GRID_D ** 1.5)
    assert abs(f["p"] - 1.5) < 1e-9 and abs(f["k"] - 3.0) < 1e-9 and abs(f["r2"] - 1.0) < 1e-9


def test_fit_two_points_hand():
    """Two points determine the line: (10, 5), (1000, 500) -> p = 1, k = 0.5."""
    f = fit_power_law([10, 1000], [5, 500])
    assert abs(f["p"] - 1.0) < 1e-12 and abs(f["k"] - 0.5) < 1e-12 and f["r2"] == pytest.approx(1.0)


def test_fit_r2_hand():
    """Logs (0,0), (1,1), (2,3) [x = e^0, e^1, e^2; y = e^0, e^1, e^3]: slope
    1.5, intercept -1/6, residuals (1/6, -1/3, 1/6): SS_res = 1/6, SS_tot =
    (4/3)^2 + (1/3)^2 + (5/3)^2 = 14/3 -> R^2 = 1 - (1/6)/(14/3) = 27/28."""
    e = math.e
    f = fit_power_law([1, e, e * e], [1, e, e ** 3])
    assert f["p"] == pytest.approx(1.5, abs=1e-12)
    assert math.log(f["k"]) == pytest.approx(-1 / 6, abs=1e-12)
    assert f["r2"] == pytest.approx(27 / 28, abs=1e-12)


def test_fit_noise_recovery():
    """Multiplicative lognormal noise (sigma 0.05) on the six grid dimensions:
    p within 0.1 of the truth and R^2 >= 0.9 over 100 seeded draws."""
    for s in range(100):
        rng = np.random.default_rng([7, s])
        p_true = rng.uniform(0.5, 2.0)
        y = 2e-3 * GRID_D ** p_true * np.exp(rng.normal(0.0, 0.05, size=GRID_D.size))
        f = fit_power_law(GRID_D, y)
        assert abs(f["p"] - p_true) <= 0.1 and f["r2"] >= 0.9


def test_fit_rejects_bad_input():
    with pytest.raises(ValueError):
        fit_power_law([1, 2], [1, 0])
    with pytest.raises(ValueError):
        fit_power_law([5, 5, 5], [1, 2, 3])
    with pytest.raises(ValueError):
        fit_power_law([1], [1])


def test_cube_generator_contract():
    x = gen.cube_cloud(500, 50, 3)
    assert x.shape == (500, 50) and x.dtype == np.float32
    assert x.min() >= 0.0 and x.max() < 1.0
    assert np.array_equal(x, gen.cube_cloud(500, 50, 3))                 # seeded
    assert not np.array_equal(x, gen.cube_cloud(500, 50, 4))             # trials differ
    assert gen.cube_eps(6) == 0.5 and gen.cube_eps(600) == pytest.approx(5.0)
    assert gen.PAPER_GRID_N == (100, 500, 1000, 2000, 5000)
    assert gen.PAPER_GRID_D == (10, 50, 100, 200, 500, 1000)


@pytest.mark.gpu
@pytest.mark.parametrize("n,D", [(100, 10), (500, 10), (1000, 50), (500, 200), (2000, 100),
                                 (500, 1000), (5000, 10)])
def test_paper_grid_cell_parity(n, D):
    import torch

    import paper_2601_01405_b200 as bm
    from tests.parity import compare

    X = gen.cube_cloud(n, D, 1)
    eps = gen.cube_eps(D)
    cov = bm.cover_build(torch.from_numpy(X).cuda(), "l2", eps)
    compare(X, "l2", eps, cov, float_path=True)
    h = bm.cover_build_host(X, "l2", eps)
    assert h.L == cov.L and h.M == cov.M and h.E == cov.E
