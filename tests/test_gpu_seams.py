"""Kernel-level entry points of the iteration's inner seams against numpy
restatements of the reference's per-op code: the prox step of update_ista / update_fista /
update_cp (solvers.py:168-225, 296-313), GroupLayout.prox (dictionary.py:290-301, via the
oracle's Layout.shrink in numpy's reduceat order), the residual (solvers.py:160-165) and the
kept-set compaction of screen_update (screening.py:104-112).

Correlations are fp64 dot products in a different summation order than numpy's BLAS (rel
1e-12); everything computed *from* the device correlations is compared bit for bit.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import ops  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from oracle import screen_oracle as so  # noqa: E402


def _setup(n, k, seed, dtype="f64"):
    D = wl.gaussian_dictionary(n, k, seed)
    if dtype == "f32":
        dic = ds.Dictionary(D.astype(np.float32), check_unit_norms=False, dtype="f32")
    elif dtype == "bf16":
        dic = ds.Dictionary(wl.bf16_round(D).reshape(D.shape), check_unit_norms=False, dtype="bf16")
    else:
        dic = ds.Dictionary(D)
    D64 = dic.as_float64()
    rng = np.random.default_rng(seed)
    theta = rng.standard_normal(n)
    point = np.where(rng.random(k) < 0.2, rng.standard_normal(k), 0.0)
    x_prev = np.where(rng.random(k) < 0.2, rng.standard_normal(k), 0.0)
    return dic, D64, theta, point, x_prev


@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
def test_corr_prox_lasso_matches_reference_step(dtype):
    dic, D, theta, point, x_prev = _setup(300, 2000, 1, dtype)
    active = np.sort(np.random.default_rng(2).choice(2000, 1500, replace=False))
    L, lam, beta = 7.3, 0.21, 0.37
    x, u, corr, (cmax, cs, ss) = ops.corr_prox(dic, active, theta, point, lam, L=L, x_prev=x_prev, beta=beta)
    ref_c = D[:, active].T @ theta
    np.testing.assert_allclose(corr[active], ref_c, rtol=1e-12, atol=1e-13 * np.max(np.abs(ref_c)))
    c = corr[active]
    xo = so.soft(point[active] - c / L, lam / L)                 # solvers.py:178
    assert np.array_equal(x[active], xo)
    assert np.array_equal(u[active], xo + beta * (xo - x_prev[active]))   # solvers.py:216-218
    rest = np.setdiff1d(np.arange(2000), active)
    assert not np.any(x[rest]) and not np.any(u[rest])
    assert cmax == float(np.max(np.abs(c)))
    d = xo - point[active]
    assert cs == pytest.approx(float(c @ d), rel=1e-12, abs=1e-14)
    assert ss == pytest.approx(float(d @ d), rel=1e-12)


def test_corr_prox_cp_step_and_empty_active():
    dic, D, theta, point, _ = _setup(200, 700, 3)
    active = np.arange(0, 700, 3)
    tau, lam = 0.05, 0.3
    x, u, corr, _ = ops.corr_prox(dic, active, theta, point, lam, tau=tau)
    assert u is None
    c = corr[active]
    assert np.array_equal(x[active], so.soft(point[active] - tau * c, lam * tau))   # solvers.py:302
    x0, _, _, red = ops.corr_prox(dic, [], theta, point, lam, L=1.0)
    assert not np.any(x0) and red == (0.0, 0.0, 0.0)
    with pytest.raises(ValueError):
        ops.corr_prox(dic, active, theta, point, lam, L=1.0, tau=1.0)


def test_corr_prox_tall_dictionary():
    dic, D, theta, point, x_prev = _setup(30011, 300, 4)
    active = np.arange(300)
    x, u, corr, _ = ops.corr_prox(dic, active, theta, point, 0.5, L=3.0, x_prev=x_prev, beta=0.5)
    np.testing.assert_allclose(corr, D.T @ theta, rtol=1e-12, atol=1e-12)
    assert np.array_equal(x, so.soft(point - corr / 3.0, 0.5 / 3.0))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_group_corr_prox_matches_group_layout(dtype):
    dic, D, theta, point, x_prev = _setup(250, 1200, 5, dtype)
    groups = [np.arange(g, g + 6) for g in range(0, 1200, 6)]
    part = ds.GroupPartition.build(dic, groups)
    active_groups = np.sort(np.random.default_rng(6).choice(200, 150, replace=False))
    L, lam, beta = 9.0, 0.4, 0.2
    x, u, corr, cn, (bound, cs, ss) = ops.group_corr_prox(dic, part, active_groups, theta, point, lam, L=L,
                                                          x_prev=x_prev, beta=beta)
    atoms = np.concatenate([groups[g] for g in active_groups])
    np.testing.assert_allclose(corr[atoms], D[:, atoms].T @ theta, rtol=1e-12, atol=1e-12)
    op = so.make_problem(D, np.zeros(250), lam, groups, part.weights, part.spectral_norms)
    lay = so.Layout(op, atoms)
    v = np.zeros(1200)
    v[atoms] = point[atoms] - corr[atoms] / L
    ref = lay.shrink(v[atoms], lam / L)                    # GroupLayout.prox (dictionary.py:290-301)
    assert np.array_equal(x[atoms], ref)
    assert np.array_equal(u[atoms], ref + beta * (ref - x_prev[atoms]))
    nc = lay.norms(corr[atoms])
    assert np.array_equal(cn, nc)
    assert bound == float(np.min(np.asarray(part.weights)[active_groups] / nc))   # screening.py:143-165
    d = ref - point[atoms]
    assert ss == pytest.approx(float(d @ d), rel=1e-12)


@pytest.mark.parametrize("dtype", ["f64", "bf16"])
def test_residual_matches_apply(dtype):
    dic, D, theta, _, _ = _setup(700, 3000, 7, dtype)
    rng = np.random.default_rng(8)
    idx = np.sort(rng.choice(3000, 333, replace=False))
    x, u = rng.standard_normal(333), rng.standard_normal(333)
    y = wl.gaussian_observation(700, 8)
    rx, ru, (qx, qu, uy) = ops.residual(dic, idx, x, y, u)
    ex, eu = D[:, idx] @ x - y, D[:, idx] @ u - y
    np.testing.assert_allclose(rx, ex, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ru, eu, rtol=1e-12, atol=1e-12)
    assert qx == pytest.approx(float(rx @ rx), rel=1e-13)
    assert qu == pytest.approx(float(ru @ ru), rel=1e-13) and uy == pytest.approx(float(ru @ y), rel=1e-12)
    r0, _, (q0, _, _) = ops.residual(dic, [], [], y)
    assert np.array_equal(r0, -y) and q0 == pytest.approx(float(y @ y), rel=1e-14)


@pytest.mark.parametrize("n", [0, 1, 1023, 1024, 1025, 300001])
def test_compact_is_order_preserving(n):
    rng = np.random.default_rng(n)
    active = np.sort(rng.choice(4 * max(n, 1), n, replace=False))
    for p in (0.0, 0.3, 1.0):
        mask = rng.random(n) < p
        assert np.array_equal(ops.compact(active, mask), active[~mask])


def test_seams_drive_one_fista_iteration_like_the_oracle():
    """corr_prox + residual + compact chained by hand reproduce the oracle's first FISTA
    iterations (fixed L, dynamic SAFE) on a c1-shaped problem."""
    w = wl.config1()
    dic = ds.Dictionary(w.D)
    L = float(np.linalg.norm(w.D, 2) ** 2 * (1 + 1e-6))
    op = so.make_problem(w.D, w.y, w.lam)
    geo = so.Geometry(op, so.lambda_max(op))
    snaps = []
    so.solve(op, so.Config(algorithm="fista", strategy="dynamic", test="safe", max_iters=5, rel_tol=1e-300, L0=L),
             hook=lambda info: snaps.append({k: np.copy(v) if isinstance(v, np.ndarray) else v
                                             for k, v in info.items()}))
    k = w.D.shape[1]
    active = np.arange(k)
    x = np.zeros(k)
    u = np.zeros(k)
    l_acc = 1.0
    for t in range(1, 6):
        theta = w.D[:, active] @ u[active] - w.y if t > 1 else -w.y
        l_new = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * l_acc ** 2))
        beta = (l_acc - 1.0) / l_new
        xn, un, corr, (cmax, _, _) = ops.corr_prox(dic, active, theta, u, w.lam, L=L, x_prev=x, beta=beta)
        l_acc = l_new
        s = snaps[t - 1]
        assert np.array_equal(s["kept"], active)
        np.testing.assert_allclose(xn[active], s["x"], rtol=1e-9, atol=1e-12)
        r, _ = geo.radius("safe", theta, corr_inf=cmax)
        mask = geo.mask("safe", r, active)
        active = ops.compact(active, mask)
        x = np.where(np.isin(np.arange(k), active), xn, 0.0)
        u = np.where(np.isin(np.arange(k), active), un, 0.0)
        supp = np.flatnonzero(x)
        rx, _, (q, _, _) = ops.residual(dic, supp, x[supp], w.y)
        assert 0.5 * q + w.lam * np.sum(np.abs(x)) == pytest.approx(s_obj(op, x), rel=1e-12)


def s_obj(op, x):
    return so.objective(op, x)
