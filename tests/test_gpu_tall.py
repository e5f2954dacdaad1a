"""Dictionaries taller than the shared-memory staging buffer (n_rows > ~27000).

The reference's Dictionary (dictionary.py:37-117) takes any N.  K1 and the setup correlations
stage theta / the correlated vector in shared memory up to ~27000 rows; taller dictionaries read
it through L2 (``theta_gl``).  Same results as the oracle: iterations, screened sets, objective.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from oracle import screen_oracle as so  # noqa: E402


def _tall(n, k, seed):
    D = wl.gaussian_dictionary(n, k, seed)
    y, _ = wl.planted_observation(D, seed, nnz=8)
    return D, y


@pytest.mark.parametrize("n", [30000, 50011])
def test_tall_correlate_apply_match_numpy(n):
    D, y = _tall(n, 600, 3)
    dic = ds.Dictionary(D)
    np.testing.assert_allclose(dic.correlate(y), D.T @ y, rtol=1e-12, atol=1e-13)
    x = np.zeros(600)
    x[::37] = np.linspace(-1, 1, x[::37].size)
    np.testing.assert_allclose(dic.apply(x), D @ x, rtol=1e-12, atol=1e-13)
    nrm = ds.operator_norm(dic, tol=1e-12, max_iters=20000)
    assert nrm == pytest.approx(float(np.linalg.norm(D, 2)), rel=1e-8)


@pytest.mark.parametrize("algo,test,ratio", [("fista", "dst3", 0.6), ("ista", "safe", 0.8), ("sparsa", "dst3", 0.7)])
def test_tall_solve_matches_oracle(algo, test, ratio):
    D, y = _tall(40000, 1200, 5)
    lam = ratio * wl.lambda_star(D, y)
    L = float(np.linalg.norm(D, 2) ** 2 * (1 + 1e-9))
    cfg = ds.SolverConfig(algorithm=algo, strategy="dynamic", test=test, max_iters=2000, rel_tol=1e-300, L0=L,
                          gap_tol=1e-8)
    res = ds.run(ds.Problem(ds.Dictionary(D), y, lam), cfg)
    ref = so.solve(so.make_problem(D, y, lam), so.Config(algorithm=algo, strategy="dynamic", test=test,
                                                         max_iters=2000, rel_tol=1e-300, L0=L, gap_tol=1e-8))
    assert res.iterations == ref.iterations
    assert np.array_equal(res.screen_state.eliminated, ref.eliminated)
    assert res.final_objective == pytest.approx(ref.final_objective, rel=1e-9)
    assert np.linalg.norm(res.x_star - ref.x_star) <= 1e-7 * max(np.linalg.norm(ref.x_star), 1e-300)
    assert res.trace.kept == ref.trace["kept"]


def test_tall_fp32_group_solve_matches_oracle():
    n, k, gs = 36000, 800, 8
    D, _ = _tall(n, k, 7)
    groups = [np.arange(g, g + gs) for g in range(0, k, gs)]
    dic = ds.Dictionary(D.astype(np.float32), check_unit_norms=False, dtype="f32")
    D64 = dic.as_float64()
    part = ds.GroupPartition.build(dic, groups)
    y = wl.bernoulli_gaussian_observation(D64, groups, 7, p=0.05)
    lam = 0.5 * wl.lambda_star(D64, y, groups, part.weights)
    L = float(np.linalg.norm(D64, 2) ** 2 * (1 + 1e-9))
    cfg = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="gst3", max_iters=2000, rel_tol=1e-300, L0=L,
                          gap_tol=1e-8)
    res = ds.run(ds.Problem(dic, y, lam, part), cfg)
    op = so.make_problem(D64, y, lam, [np.asarray(g) for g in groups], part.weights, part.spectral_norms)
    ref = so.solve(op, so.Config(algorithm="fista", strategy="dynamic", test="gst3", max_iters=2000,
                                 rel_tol=1e-300, L0=L, gap_tol=1e-8))
    assert res.iterations == ref.iterations
    assert np.array_equal(res.screen_state.eliminated, ref.eliminated)
    assert res.final_objective == pytest.approx(ref.final_objective, rel=1e-9)
