"""Engine robustness on the GPU:

* the reference's error paths through ``run()`` (tests/error_cases.py, reference outcomes in
  tests/golden/error_cases.json): FloatingPointError (solvers.py:157-159, 186-187),
  RuntimeError for the radius guard (screening.py:199-205) and the degenerate GST3 normal
  (screening.py:245-246), plus the overflow run the reference completes with +inf objectives;
* device caches keyed by content: two observations solved on one Dictionary object, and two
  partitions with the same groups but different weights, each against the oracle.
"""

import json
import os
import warnings

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from oracle import screen_oracle as so  # noqa: E402
from tests.error_cases import CASES  # noqa: E402

with open(os.path.join(os.path.dirname(__file__), "golden", "error_cases.json")) as fh:
    GOLD = json.load(fh)


@pytest.mark.parametrize("name,build", CASES, ids=[c[0] for c in CASES])
def test_engine_error_paths_match_reference(name, build):
    c = build()
    ref = GOLD[name]
    dic = ds.Dictionary(c["D"], check_unit_norms=c["check_unit_norms"])
    part = ds.GroupPartition.build(dic, c["groups"], weights=c["weights"]) if c["groups"] is not None else None
    prob = ds.Problem(dic, c["y"], c["lam"], part)
    cfg = ds.SolverConfig(**c["cfg"])
    if ref["outcome"] == "ok":
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = ds.run(prob, cfg)
        assert res.iterations == ref["iterations"]
        assert res.trace.objective == ref["objective"]
        assert bool(np.all(np.isfinite(res.x_star))) == ref["x_finite"]
        assert float(np.max(np.abs(res.x_star))) == pytest.approx(ref["x_absmax"], rel=1e-12)
        return
    exc = {"FloatingPointError": FloatingPointError, "RuntimeError": RuntimeError}[ref["outcome"]]
    with pytest.raises(exc):
        ds.run(prob, cfg)


def _oracle(D, y, lam, cfg, groups=None, weights=None, snorms=None):
    return so.solve(so.make_problem(D, y, lam, groups, weights, snorms),
                    so.Config(algorithm=cfg.algorithm, strategy=cfg.strategy, test=cfg.test,
                              max_iters=cfg.max_iters, rel_tol=cfg.rel_tol, L0=cfg.L0, gap_tol=cfg.gap_tol))


def _check(res, ref):
    assert res.iterations == ref.iterations
    assert np.array_equal(res.screen_state.eliminated, ref.eliminated)
    np.testing.assert_allclose(res.final_objective, ref.final_objective, rtol=1e-10)
    assert np.linalg.norm(res.x_star - ref.x_star) <= 1e-8 * max(np.linalg.norm(ref.x_star), 1e-300)


def test_two_observations_on_one_dictionary():
    D = wl.correlated_dictionary(200, 1000, 4)
    dic = ds.Dictionary(D)
    L = float(np.linalg.norm(D, 2) ** 2 * (1 + 1e-9))
    cfg = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="dst3", max_iters=3000, rel_tol=1e-300,
                          L0=L, gap_tol=1e-8)
    seen = []
    for seed, ratio in ((4, 0.6), (5, 0.4), (4, 0.6)):     # (4, 0.6) again after (5, 0.4): cache reuse
        y, _ = wl.planted_observation(D, seed, nnz=8)
        lam = ratio * wl.lambda_star(D, y)
        res = ds.run(ds.Problem(dic, y, lam), cfg)
        _check(res, _oracle(D, y, lam, cfg))
        seen.append(res.final_objective)
    assert seen[0] != seen[1] and seen[0] == seen[2]


def test_partitions_with_equal_groups_and_different_weights():
    D = wl.gaussian_dictionary(150, 600, 6)
    groups = [np.arange(g, g + 6) for g in range(0, 600, 6)]
    dic = ds.Dictionary(D)
    L = float(np.linalg.norm(D, 2) ** 2 * (1 + 1e-9))
    cfg = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="gst3", max_iters=3000, rel_tol=1e-300,
                          L0=L, gap_tol=1e-8)
    y = wl.gaussian_observation(150, 6)
    base = ds.GroupPartition.build(dic, groups)
    for scale in (1.0, 1.7, 1.0):
        w = np.sqrt(6.0) * scale * (1.0 + 0.1 * (np.arange(100) % 3))
        part = ds.GroupPartition.build(dic, groups, weights=w, spectral_norms=base.spectral_norms)
        lam = 0.5 * wl.lambda_star(D, y, groups, w)
        res = ds.run(ds.Problem(dic, y, lam, part), cfg)
        _check(res, _oracle(D, y, lam, cfg, groups, w, base.spectral_norms))
