"""BASELINE-config parity at full size (c1, c2 sweep, c3) and a c4 proxy.

Checks per BASELINE.json north_star (oracle/parity.py): (1) safety against a
certified coordinate-descent solution, (2) screened sets equal up to atoms within
1e-9 of the test threshold at some iteration (margins from the oracle's per-t
radius), (3) objective (final and per iteration) and x within rel 1e-6 (fp64) /
1e-4 (fp32), (4) equal iteration counts to the gap tolerance.  The full-size c4
run is checked against the reference itself in tests/test_gpu_c4_full.py.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from oracle import parity  # noqa: E402
from oracle import screen_oracle as so  # noqa: E402

_L = {}


def _spec_L(dic):
    key = id(dic)
    if key not in _L:
        nrm = ds.operator_norm(dic, tol=1e-12, max_iters=20000)
        _L[key] = nrm * nrm * (1.0 + 1e-6)
    return _L[key]


def _compare(w, dic, part=None, x_rtol=1e-6):
    """The four north_star checks (oracle/parity.py) on one BASELINE workload."""
    prob = ds.Problem(dic, w.y, w.lam, part)
    L = _spec_L(dic)
    cfg = ds.SolverConfig(algorithm=w.algorithm, strategy="dynamic", test=w.test, max_iters=w.max_iters,
                          rel_tol=1e-300, L0=L, gap_tol=w.gap_tol)
    res = ds.run(prob, cfg)
    D64 = dic.as_float64()
    op = so.make_problem(D64, w.y, w.lam, w.groups, None if part is None else part.weights,
                         None if part is None else part.spectral_norms)
    rec = parity.RadiusRecorder()
    ref = so.solve(op, so.Config(algorithm=w.algorithm, strategy="dynamic", test=w.test,
                                 max_iters=w.max_iters, rel_tol=1e-300, L0=L, gap_tol=w.gap_tol,
                                 norm_aware=dic.norm_aware), hook=rec)
    # 4. iteration counts to the gap tolerance
    assert res.stop_reason == "gap"
    assert res.iterations == ref.iterations, (res.iterations, ref.iterations)
    # 3. objective and iterate
    np.testing.assert_allclose(res.final_objective, ref.final_objective, rtol=x_rtol)
    assert parity.rel(res.x_star, ref.x_star) <= x_rtol, parity.rel(res.x_star, ref.x_star)
    np.testing.assert_allclose(res.trace.objective, ref.trace["objective"], rtol=x_rtol)
    # 2. screened sets: equal up to units within 1e-9 of the test threshold at some iteration
    ok, diff, margins = parity.screened_sets_agree(op, w.test, res.screen_state.eliminated, ref.eliminated,
                                                   rec.radius, dic.norm_aware)
    assert ok, (diff[:10], margins[:10])
    if diff.size == 0:
        assert res.trace.kept == ref.trace["kept"]
    # 1. safety against the certified coordinate-descent solution (trivial when nothing is screened)
    safe, _ = parity.certified_safe(op, res.screen_state.eliminated)
    assert safe
    return res, ref


def test_c1_ista_dst3():
    w = wl.config1()
    _compare(w, ds.Dictionary(w.D))


@pytest.mark.parametrize("ratio", [0.1, 0.3, 0.5, 0.7, 0.9])
@pytest.mark.parametrize("test", ["dst3", "safe"])
def test_c2_fista_sweep(ratio, test):
    """BASELINE c2: all five lambda/lambda_* ratios x {SAFE, DST3}."""
    w = wl.config2(ratio=ratio, test=test)
    _compare(w, _c2_dic(w.D))


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
    _compare(w, dic, part)


def test_c4_proxy_fp32():
    """1024 x 32768 fp32 proxy of c4; oracle in fp64 on the upcast dictionary."""
    D = wl.gaussian_dictionary_f32(1024, 32768, 0)
    y = wl.gaussian_observation(1024, 0)
    lam = 0.2 * float(np.max(np.abs(D.astype(np.float64).T @ y)))
    w = wl.Workload("c4proxy", D, y, lam, algorithm="fista", test="dst3", gap_tol=1e-5, dtype="f32")
    dic = ds.Dictionary(D, check_unit_norms=False, dtype="f32")
    _compare(w, dic, x_rtol=1e-4)
