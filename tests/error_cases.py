"""Inputs that drive the reference's error paths (shared by the golden generator and the tests).

Each case: (name, build) where build() -> dict(D, y, lam, groups|None, weights|None,
check_unit_norms, cfg) with cfg the SolverConfig fields.  The reference outcomes live in
tests/golden/error_cases.json (tests/golden/make_error_golden.py ran screenlab itself):
* FloatingPointError "non-finite iterate" (solvers.py:157-159): SpaRSA from L0 = 1e-300 with
  the BB floor lowered to 1e-300; TwIST with step 1e300;
* FloatingPointError "backtracking failed" (solvers.py:186-187): ISTA on an unchecked
  dictionary scaled by 1e200 (every candidate overflows);
* an ISTA run from L0 = 1e-300 that the reference *completes* (finite iterates of size 1e299,
  every objective +inf: the majorisation test compares inf <= inf);
* RuntimeError radius guard (screening.py:199-205): DST3 on an unchecked fp64 dictionary whose
  columns have norm 2 (the reference's unit-atom DST3 radius goes negative), ISTA and FISTA;
* RuntimeError degenerate GST3 normal (screening.py:245-246): group weights 1e-170, so
  lambda_* ~ 1e170 and the tangent normal D_g D_g^T y / lambda_* underflows to exactly zero.
"""

import numpy as np

from paper_1412_4080_b200 import workloads as wl


def _base():
    return wl.gaussian_dictionary(20, 50, 1), wl.gaussian_observation(20, 1)


def _lstar(D, y):
    return float(np.max(np.abs(D.T @ y)))


def _case(D, y, lam, cfg, groups=None, weights=None, check=True):
    return dict(D=np.asfortranarray(D), y=y, lam=float(lam), groups=groups, weights=weights,
                check_unit_norms=check, cfg=cfg)


def sparsa_overflow():
    D, y = _base()
    return _case(D, y, 0.5 * _lstar(D, y), dict(algorithm="sparsa", max_iters=50, L0=1e-300, bb_L_min=1e-300))


def twist_overflow():
    D, y = _base()
    return _case(D, y, 0.5 * _lstar(D, y), dict(algorithm="twist", max_iters=50, twist_step=1e300))


def ista_backtrack_fail():
    D, y = _base()
    D = D * 1e200
    return _case(D, y, 0.5 * _lstar(D, y), dict(algorithm="ista", max_iters=50), check=False)


def ista_inf_objective():
    D, y = _base()
    return _case(D, y, 0.5 * _lstar(D, y), dict(algorithm="ista", max_iters=50, L0=1e-300))


def radius_guard_ista():
    D, y = _base()
    D = 2.0 * D
    L = float(np.linalg.norm(D, 2) ** 2)
    return _case(D, y, 0.5 * _lstar(D, y), dict(algorithm="ista", strategy="dynamic", test="dst3",
                                                max_iters=200, L0=L), check=False)


def radius_guard_fista():
    c = radius_guard_ista()
    c["cfg"]["algorithm"] = "fista"
    return c


def gst3_degenerate():
    D, y = _base()
    groups = [np.arange(i, i + 5) for i in range(0, 50, 5)]
    w = np.full(10, 1e-170)
    lstar = max(float(np.linalg.norm(D[:, g].T @ y)) / 1e-170 for g in groups)
    return _case(D, y, 0.5 * lstar, dict(algorithm="fista", strategy="dynamic", test="gst3", max_iters=5, L0=1.0),
                 groups=groups, weights=w)


CASES = [("sparsa_overflow", sparsa_overflow), ("twist_overflow", twist_overflow),
         ("ista_backtrack_fail", ista_backtrack_fail), ("ista_inf_objective", ista_inf_objective),
         ("radius_guard_ista", radius_guard_ista), ("radius_guard_fista", radius_guard_fista),
         ("gst3_degenerate", gst3_degenerate)]
