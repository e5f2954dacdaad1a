"""The tiled K1 path (columns of 5..16 segments of 256 rows: atom-quad x row-segment items,
fixed-order segment sums) against the CPU oracle: fp64 and fp32 Lasso, groups of mixed sizes
(up to the 64-atom shared-memory limit of the tiled group update), and a partition with one
group wider than 64 atoms (per-warp column path).  Screening fires in every case, so the
identity-list shortcut is also left behind mid-solve."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from oracle import screen_oracle as so  # noqa: E402


def _run(D, y, lam, groups=None, dtype="f64", algo="fista", test="dst3", rtol=1e-9, gap_tol=1e-7):
    dic = ds.Dictionary(D, check_unit_norms=(dtype == "f64"), dtype=dtype)
    part = ds.GroupPartition.build(dic, groups) if groups is not None else None
    D64 = dic.as_float64()
    L = float(np.linalg.norm(D64, 2) ** 2 * (1 + 1e-9))
    cfg = ds.SolverConfig(algorithm=algo, strategy="dynamic", test=test, max_iters=3000, rel_tol=1e-300,
                          L0=L, gap_tol=gap_tol)
    res = ds.run(ds.Problem(dic, y, lam, part), cfg)
    op = so.make_problem(D64, y, lam, groups, None if part is None else part.weights,
                         None if part is None else part.spectral_norms)
    ref = so.solve(op, so.Config(algorithm=algo, strategy="dynamic", test=test, max_iters=3000, rel_tol=1e-300,
                                 L0=L, gap_tol=gap_tol, norm_aware=dic.norm_aware))
    # gap 1e-7: reached well before the objective stalls to the last bit (rel_tol 1e-300 stops on
    # bitwise-equal consecutive objectives, where 1-ulp summation differences decide)
    assert res.stop_reason == "gap"
    assert res.iterations == ref.iterations
    assert np.array_equal(res.screen_state.eliminated, ref.eliminated)
    assert ref.eliminated.size > 0
    np.testing.assert_allclose(res.final_objective, ref.final_objective, rtol=rtol)
    assert np.linalg.norm(res.x_star - ref.x_star) <= 1e-6 * max(np.linalg.norm(ref.x_star), 1e-300)
    return res


@pytest.mark.parametrize("n", [1300, 4000, 5000])   # 5000: > 16 segments, per-warp column path
def test_tiled_lasso_f64(n):
    D = wl.correlated_dictionary(n, 3000, 11)
    y, _ = wl.planted_observation(D, 11, nnz=12)
    _run(D, y, 0.6 * wl.lambda_star(D, y))


@pytest.mark.parametrize("n", [1300, 8192])          # 8192 (c4 rows): per-warp column path
def test_tiled_lasso_f32(n):
    D = wl.correlated_dictionary(n, 3000, 12).astype(np.float32)
    y, _ = wl.planted_observation(D.astype(np.float64), 12, nnz=12)
    _run(D, y, 0.6 * wl.lambda_star(D.astype(np.float64), y), dtype="f32", rtol=1e-6)


def _mixed_groups(k, seed, wide=None):
    rng = np.random.default_rng(seed)
    sizes = []
    while sum(sizes) < k:
        sizes.append(int(rng.integers(1, 41)))
    sizes[-1] -= sum(sizes) - k
    if sizes[-1] <= 0:
        sizes.pop()
        sizes[-1] += k - sum(sizes)
    if wide:
        sizes = [wide] + sizes
        sizes[-1] -= wide
        while sizes[-1] <= 0:
            extra = sizes.pop()
            sizes[-1] += extra
    ptr = np.concatenate(([0], np.cumsum(sizes)))
    return [np.arange(ptr[g], ptr[g + 1]) for g in range(len(sizes))]


@pytest.mark.parametrize("wide", [None, 80], ids=["sizes-1-40", "one-group-of-80"])
def test_tiled_groups(wide):
    D = wl.correlated_dictionary(1300, 2400, 13)
    groups = _mixed_groups(2400, 13, wide)
    y, _ = wl.planted_observation(D, 13, nnz=15)
    corr = D.T @ y
    w = np.sqrt([g.size for g in groups])
    lam = 0.7 * max(np.linalg.norm(corr[g]) / wg for g, wg in zip(groups, w))
    _run(D, y, lam, groups=groups, test="gst3")


def test_rows_beyond_shared_memory_theta_are_solved():
    """Taller than the shared-memory theta buffer (8 bytes per row): theta is read through L2
    and the solve matches the oracle (a degenerate identity-block dictionary; tests/test_gpu_tall.py
    covers Gaussian tall dictionaries)."""
    D = np.zeros((30000, 8))
    D[np.arange(8), np.arange(8)] = 1.0
    y = np.zeros(30000)
    y[:8] = np.linspace(1.0, 0.2, 8)
    y /= np.linalg.norm(y)
    cfg = ds.SolverConfig(algorithm="ista", strategy="dynamic", test="dst3", max_iters=5, L0=1.0)
    res = ds.run(ds.Problem(ds.Dictionary(D), y, 0.5), cfg)
    ref = so.solve(so.make_problem(D, y, 0.5), so.Config(algorithm="ista", strategy="dynamic", test="dst3",
                                                          max_iters=5, L0=1.0))
    assert res.iterations == ref.iterations
    assert np.array_equal(res.screen_state.eliminated, ref.eliminated)
    np.testing.assert_allclose(res.x_star, ref.x_star, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("algo", ["fista", "ista"])
def test_wide_k2_rounds(algo):
    """More than 256 active units per K2 CTA (80000 columns over 296 CTAs): the 4-units-per-
    thread K2 rounds while the list is the identity, the classic rounds after screening."""
    D = wl.correlated_dictionary(256, 80000, 21)
    y, _ = wl.planted_observation(D, 21, nnz=8)
    _run(D, y, 0.85 * wl.lambda_star(D, y), algo=algo, gap_tol=1e-6)
