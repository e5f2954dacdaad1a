"""Pin the CPU oracle against golden vectors produced by the reference itself."""

import numpy as np
import pytest

from oracle import screen_oracle as so
from tests.golden_cases import kernel_cases, load

CASES = load()


def _problem(c):
    return so.make_problem(c["D"], c["y"], c["lam"], c["groups"], c["weights"], c["snorms"])


def _cfg(c):
    d = dict(c["cfg"])
    return so.Config(**d)


@pytest.mark.parametrize("idx", range(len(CASES)), ids=[f"{c['name']}-{i}" for i, c in enumerate(CASES)])
def test_oracle_matches_reference_run(idx):
    c = CASES[idx]
    p = _problem(c)
    res = so.solve(p, _cfg(c))
    ref = c["ref"]
    assert res.iterations == ref["iterations"]
    assert np.array_equal(res.eliminated, ref["eliminated"])
    assert np.array_equal(np.array(res.trace["kept"]), ref["kept"])
    assert np.array_equal(np.array(res.trace["nnz"]), ref["nnz"])
    assert np.array_equal(np.array(res.trace["flops"]), ref["flops"])
    scale = max(1.0, float(np.max(np.abs(ref["x_star"]), initial=0.0)))
    assert np.max(np.abs(res.x_star - ref["x_star"]), initial=0.0) <= 1e-12 * scale
    np.testing.assert_allclose(res.trace["objective"], ref["objective"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(res.trace["gap"], ref["gap"], rtol=1e-9, atol=1e-13)
    assert res.final_objective == pytest.approx(ref["final_objective"], rel=1e-12, abs=1e-14)


def test_lambda_max_matches_reference():
    seen = set()
    for c in CASES:
        if c["pid"] in seen:
            continue
        seen.add(c["pid"])
        lm = so.lambda_max(_problem(c))
        assert lm.value == pytest.approx(c["lmax"], rel=1e-14)
        if c["kind"] == "lasso":
            assert lm.index == c["lmax_index"]
        else:
            assert lm.group == c["lmax_group"]


def test_operator_norm_matches_reference():
    seen = set()
    for c in CASES:
        if c["pid"] in seen or c["D"].size > 5000:
            continue
        seen.add(c["pid"])
        assert so.operator_norm(c["D"]) == pytest.approx(c["op_norm"], rel=1e-12)


def test_per_op_golden():
    k = kernel_cases()
    for i in range(20):
        out = so.soft(k[f"prox_l1_{i}__v"], float(k[f"prox_l1_{i}__t"]))
        assert np.array_equal(out, k[f"prox_l1_{i}__out"])
    groups = [np.arange(0, 4), np.arange(4, 7), np.arange(7, 12)]
    D = np.eye(12)
    p = so.make_problem(D, np.eye(12)[0], 0.5, groups, snorms=np.ones(3))
    lay = so.Layout(p, np.arange(12))
    for i in range(10):
        out = lay.shrink(k[f"prox_group_{i}__v"], float(k[f"prox_group_{i}__t"]))
        assert np.array_equal(out, k[f"prox_group_{i}__out"])
    for i in range(10):
        assert so.operator_norm(k[f"opnorm_{i}__D"]) == pytest.approx(float(k[f"opnorm_{i}__out"]), rel=1e-12)


def test_known_answers():
    # identity instance: x* = (0.2, 0), F = 0.48 (reference tests/test_solvers.py:229-235)
    p = so.make_problem(np.eye(2), np.array([1.0, 0.0]), 0.8)
    r = so.solve(p, so.Config(algorithm="ista", strategy="dynamic", test="dst3", max_iters=200, rel_tol=1e-12))
    assert np.allclose(r.x_star, [0.2, 0.0], atol=1e-9)
    assert r.final_objective == pytest.approx(0.48, abs=1e-9)
    geo = so.Geometry(p, so.lambda_max(p))
    # SAFE centre (1.25, 0), r = 0.25 (tests/test_screening.py:96-100)
    rad, _ = geo.radius("safe", p.y, corr_inf=1.0)
    assert rad == pytest.approx(0.25)
    # DST3 radius 0, mask [F, T] (tests/test_screening.py:128-133)
    rad, _ = geo.radius("dst3", p.y, corr_inf=1.0)
    assert rad == pytest.approx(0.0, abs=1e-12)
    assert geo.mask("dst3", rad, np.arange(2)).tolist() == [False, True]
    # dual scaling mu = 1, -1, 1/0.8 (tests/test_screening.py:14-29)
    assert so.dual_scale_lasso(p, p.y, 1.0)[0] == pytest.approx(1.0)
    assert so.dual_scale_lasso(p, -p.y, 1.0)[0] == pytest.approx(-1.0)
    assert so.dual_scale_lasso(p, p.y, 0.0)[0] == pytest.approx(1.25)
    # flops worked values (tests/test_instrument.py:11-16)
    assert so.flops_iteration("lasso", "none", 10, 5, 10, 2) == 105
    assert so.flops_iteration("lasso", "dynamic", 10, 5, 6, 2) == 101
    assert so.flops_iteration("group", "dynamic", 10, 5, 6, 2, 3) == 122


def test_gap_stop_hits_first_crossing():
    for c in CASES:
        if not c["name"].startswith("c2mini") or c["cfg"]["algorithm"] != "fista":
            continue
        gaps = c["ref"]["gap"]
        hit = np.flatnonzero(gaps <= 1e-6)
        if not hit.size:
            continue
        cfg = _cfg(c)
        cfg.gap_tol = 1e-6
        res = so.solve(_problem(c), cfg)
        assert res.iterations == hit[0] + 1
