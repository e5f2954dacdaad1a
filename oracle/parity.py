"""The four BASELINE parity checks (north_star; SURVEY §8(c) "Parity checks") made concrete.

TEST INFRASTRUCTURE ONLY (imported by ``tests/``, never by the product package).  Given a GPU
result (``SolveResult`` from ``paper_1412_4080_b200.run``) and an oracle run of the same
problem (``screen_oracle.solve`` with a hook that records the per-iteration test radius):

1. *safety*: no screened atom is nonzero in a certified reference solution
   (``verify_screen_safety`` after ``solve_reference(p, 1e-10)``, reference oracle.py:44-139);
2. *screened-set agreement*: the symmetric difference of the eliminated sets contains only
   atoms whose test margin ``|v_i - rho_t - 1e-12|`` lies within 1e-9 of the threshold at some
   iteration t of the oracle run (``test_sphere_lasso`` screening.py:351-359 with
   ``SCREEN_MARGIN`` screening.py:40; groups: the group margin of ``test_sphere_group``
   screening.py:391-404);
3. *objective and iterate*: relative differences within 1e-6 (fp64) / 1e-4 (fp32);
4. *iteration counts* to the gap tolerance are equal.
"""

from __future__ import annotations

import numpy as np

from . import screen_oracle as so

MARGIN_TOL = 1e-9


class RadiusRecorder:
    """Oracle hook recording the test radius of every iteration (and the active set size)."""

    def __init__(self):
        self.radius = []
        self.kept = []

    def __call__(self, info):
        self.radius.append(float(info["radius"]))
        self.kept.append(int(info["kept"].size))


def unit_test_values(prob, test, norm_aware=False, lmax=None):
    """Per-unit test value v such that a unit is screened at radius r iff v - r > 1e-12.

    Lasso SAFE/DST3: v_i = 1 - |cc_i| (norm-aware: divided by ||a_i||); group GSAFE/GST3:
    v_g = (w_g - ||D_g^T cc||) / ||D_g||.  Returns (values, unit_of_atom or None)."""
    lm = lmax if lmax is not None else so.lambda_max(prob)
    geo = so.Geometry(prob, lm, norm_aware)
    if prob.kind == so.LASSO:
        if test not in (so.SAFE, so.DST3):
            raise ValueError("margins are defined for the sphere tests")
        cc = geo.safe_cc if test == so.SAFE else geo.dst3_cc
        v = 1.0 - np.abs(cc)
        if geo.norms is not None:
            v = v / geo.norms
        return v, None
    cn = geo.center_group_norms(test)
    v = (prob.weights - cn) / prob.snorms
    gof = np.empty(prob.k, dtype=np.int64)
    for gid, g in enumerate(prob.groups):
        gof[g] = gid
    return v, gof


def margin_ok(values, radii, units, tol=MARGIN_TOL):
    """True iff every unit in `units` had |v - rho_t - 1e-12| <= tol for some recorded t."""
    units = np.asarray(units, dtype=np.int64)
    if units.size == 0:
        return True, np.empty(0)
    r = np.asarray([x for x in radii if np.isfinite(x)])
    if r.size == 0:
        return False, np.full(units.size, np.inf)
    m = np.min(np.abs(values[units][:, None] - r[None, :] - so.SCREEN_MARGIN), axis=1)
    return bool(np.all(m <= tol)), m


def screened_sets_agree(prob, test, elim_gpu, elim_ref, radii, norm_aware=False, tol=MARGIN_TOL):
    """Check 2: symmetric difference only at near-threshold units.  Returns (ok, diff, margins)."""
    diff = np.setxor1d(np.asarray(elim_gpu, np.int64), np.asarray(elim_ref, np.int64))
    if diff.size == 0:
        return True, diff, np.empty(0)
    values, gof = unit_test_values(prob, test, norm_aware)
    units = diff if gof is None else np.unique(gof[diff])
    ok, m = margin_ok(values, radii, units, tol)
    return ok, diff, m


def certified_safe(prob, eliminated, gap_tol=1e-10):
    """Check 1 (reference oracle.py:128-139).  Nothing screened is trivially safe; otherwise
    coordinate descent to a certified gap <= 1e-10 and |x_ref[eliminated]| <= 1e-9."""
    eliminated = np.asarray(eliminated, dtype=np.int64)
    if eliminated.size == 0:
        return True, 0.0
    x_ref, gap = so.cd_solve(prob, gap_tol)
    if gap > 1e-10:
        raise ValueError("reference solution is not certified tightly enough")
    return so.screen_is_safe(x_ref, eliminated), gap


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
