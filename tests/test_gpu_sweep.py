"""GPU-resident lambda sweep (cli._bench_seed restated on the device engine) vs the oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import instrument as ins  # noqa: E402
from paper_1412_4080_b200 import sweep as sw  # noqa: E402
from oracle import screen_oracle as so  # noqa: E402


def test_sweep_rows_match_oracle():
    rng = np.random.default_rng(7)
    D = rng.standard_normal((120, 400))
    D /= np.linalg.norm(D, axis=0)
    y = D[:, [3, 50, 77]] @ np.array([1.0, -0.7, 0.4]) + 0.05 * rng.standard_normal(120)
    y /= np.linalg.norm(y)
    dic = ds.Dictionary(D)
    plan = sw.SweepPlan([0.3, 0.8], algorithms=["ista", "fista"], tests=["safe", "dst3"], max_iters=300,
                        rel_tol=1e-9)
    results = []
    rows = sw.sweep(dic, y, plan, seed=3, results=results)
    assert len(rows) == 2 * 2 * (1 + 2 + 2)
    lmax = ds.lambda_max(ds.Problem(dic, y, 1.0)).value
    for row, res in zip(rows, results):
        seed, algo, strategy, test, ratio, iters, flops, t, obj, frac = row
        assert seed == 3 and t > 0
        ref = so.solve(so.make_problem(D, y, ratio * lmax),
                       so.Config(algorithm=algo, strategy=strategy, test=None if test == "-" else test,
                                 max_iters=plan.max_iters, rel_tol=plan.rel_tol, L0=1.0))
        assert iters == ref.iterations, row
        assert flops == ref.trace["flops"][-1], row
        assert frac == pytest.approx(ref.eliminated.size / D.shape[1]), row
        assert obj == pytest.approx(ref.final_objective, rel=1e-9), row
    # the paper's normalized metrics from one (none, static, dynamic) triple of the sweep
    tri = {r[2]: res.trace for r, res in zip(rows, results) if r[1] == "fista" and r[4] == 0.8 and r[3] in ("-", "dst3")}
    m = ins.normalized_metrics(tri["none"], tri["static"], tri["dynamic"])
    assert 0 < m.flops_dynamic_ratio <= 1.0 and 0 < m.flops_static_ratio <= 1.0 + 1e-12
