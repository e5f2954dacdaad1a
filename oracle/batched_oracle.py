"""CPU oracle for the batched bf16 path (BASELINE config 5).

TEST INFRASTRUCTURE ONLY (imported by ``tests/`` and ``bench.py``'s reference leg, never by the
product package).

Config 5 is specified as "bf16-in / fp32-accumulate": the shared dictionary is bf16 and the
per-iteration contraction ``D^T Theta`` takes bf16 operands.  ``screen_oracle.solve`` is the
reference's fp64 algorithm (``solvers.run`` with FISTA, ``solvers.py:207-225``, and the
dynamic DST3 test, ``screening.py:263-296``); it cannot agree with a bf16-operand solve to
better than the bf16 rounding of theta lets it (~1e-2 in the objective after 100 iterations,
measured below).  ``solve_bf16`` restates the same FISTA iteration with exactly the roundings
the config prescribes, everything else in fp64:

* theta_t = D u_t - y in fp64 (``solvers.py:212``), then rounded to bf16 (round to nearest
  even, straight from fp64) -- the GEMM operand;  ``splits=2`` adds the bf16 rounding of the
  remainder as a second term (theta_hi + theta_lo);
* c_t = D_A^T theta~_t, accumulated in fp64 (the device accumulates in fp32: the only
  arithmetic difference left between this oracle and the GPU, apart from fp32 storage of the
  test centres, covered by the test slack below);
* dual scaling (``screening.py:115-140``) with the correlation bound inflated by a rigorous
  bound on the operand error, ``max|c~| + err_rel ||theta||`` -- a bound >= the exact
  ``max|D_A^T theta|``, so the scaled point is dual feasible for the *unrounded* problem and the
  test stays safe;
* r_SAFE^2 = ||y/lam - mu theta||^2 and the DST3 radius with the norm-aware normal
  ``a*/||a*||`` (``screen_oracle.Geometry(norm_aware=True)``; at unit norms the reference's
  ``screening.py:221-231``); the sphere test ``(1-|cc_i|)/||a_i|| - rho > 1e-12 + slack``
  (``screening.py:351-359``), applied before the prox of the same iteration (screened atoms
  take no candidate: the reference's drop-and-recompute, ``solvers.py:480-488``, gives the
  same iterate);
* fixed step 1/L (BASELINE: step 1/||D||^2; the reference's backtracking test accepts L at
  once when L >= ||D||^2), FISTA momentum ``solvers.py:216-218``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import screen_oracle as so

TEST_SLACK = 1e-6           # extra test margin of the device (its centre correlations are fp32)


def bf16_rn(v):
    """Round fp64 values to the nearest bf16 (ties to even) directly from fp64, as
    ``__double2bfloat16`` does; returned as fp64.  (Finite, normal-range inputs.)"""
    v = np.ascontiguousarray(v, dtype=np.float64)
    b = v.view(np.uint64)
    lsb = (b >> np.uint64(45)) & np.uint64(1)
    r = (b + np.uint64((1 << 44) - 1) + lsb) >> np.uint64(45) << np.uint64(45)
    return r.view(np.float64)


def err_rel(n_rows, splits):
    """The device's bound on |c~ - c| / ||theta|| (dscr_batched.cu, dscr_batched_create):
    bf16 rounding of theta (2^-8 relative per element, one term; 1.6e-5 with two) plus the
    fp32 accumulation over n_rows products."""
    return (0.00391 if splits == 1 else 1.6e-5) + 2.0 * n_rows * 5.96e-8


@dataclass
class Bf16Result:
    x: np.ndarray
    objective: float
    eliminated: np.ndarray
    kept: int
    trace: dict = field(default_factory=dict)


def solve_bf16(D, y, lam, L, iterations, splits=1, test="dst3", slack=TEST_SLACK, hook=None):
    """FISTA with dynamic SAFE/DST3 screening at the config-5 operand precision (see module doc).

    ``D`` is the fp64 upcast of the bf16 dictionary.  Returns the iterate, the final objective,
    the eliminated atoms and a per-iteration trace (objective, radius, kept).  ``hook`` gets
    ``{"t", "radius", "kept"}`` before each iteration's reduction."""
    n, k = D.shape
    prob = so.make_problem(D, y, lam)
    lm = so.lambda_max(prob)
    if lam > lm.value:
        return Bf16Result(np.zeros(k), 0.5 * float(y @ y), np.arange(k), 0, {})
    geo = so.Geometry(prob, lm, norm_aware=True)
    if test == "safe":
        values = (1.0 - np.abs(geo.safe_cc)) / geo.norms
        shift_sq = 0.0
    else:
        values = (1.0 - np.abs(geo.dst3_cc)) / geo.norms
        shift_sq = geo.shift ** 2 / geo.star_norm_sq
    er = err_rel(n, splits)
    DT = np.ascontiguousarray(D.T)

    def apply(v):                       # D v for a sparse v, fp64
        nz = np.flatnonzero(v)
        return D[:, nz] @ v[nz]

    active = np.ones(k, dtype=bool)
    x = np.zeros(k)
    u = np.zeros(k)
    l_acc = 1.0
    tr = {"objective": [], "radius": [], "kept": [], "gap": []}
    for t in range(1, iterations + 1):
        theta = apply(u) - y
        tt = bf16_rn(theta)
        if splits > 1:
            tt = tt + bf16_rn(theta - tt)
        c = np.where(active, DT @ tt, 0.0)
        sq = float(theta @ theta)
        cinf = float(np.max(np.abs(c[active]), initial=0.0)) + er * np.sqrt(sq)
        bound = np.inf if cinf == 0.0 else 1.0 / cinf
        mu = float(np.clip(float(theta @ y) / (lam * sq), -bound, bound)) if sq != 0.0 else 0.0
        diff = y / lam - mu * theta
        rsq = float(diff @ diff)
        if test == "safe":
            rho = float(np.sqrt(rsq))
        else:
            arg = rsq - shift_sq
            if arg < -so.RADIUS_GUARD:
                raise RuntimeError(f"squared screening radius fell to {arg!r}")
            rho = float(np.sqrt(max(arg, 0.0)))
        if test != "off":
            active &= ~(values - rho > so.SCREEN_MARGIN + slack)
        if hook is not None:
            hook({"t": t, "radius": rho, "kept": int(active.sum())})
        cand = np.where(active, so.soft(u - c / L, lam / L), 0.0)
        l_new = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * l_acc ** 2))
        u = np.where(active, cand + ((l_acc - 1.0) / l_new) * (cand - x), 0.0)
        l_acc = float(l_new)
        x = cand
        r = apply(x) - y
        f = 0.5 * float(r @ r) + lam * float(np.sum(np.abs(x)))
        tr["objective"].append(f)
        tr["radius"].append(rho)
        tr["kept"].append(int(active.sum()))
        tr["gap"].append(f - 0.5 * float(y @ y) + 0.5 * lam * lam * rsq)
    return Bf16Result(x, tr["objective"][-1], np.flatnonzero(~active), int(active.sum()), tr)


def screen_values(D, y, lam, test="dst3"):
    """Per-atom test values v_i (screened at radius rho iff v_i - rho > margin)."""
    prob = so.make_problem(D, y, lam)
    geo = so.Geometry(prob, so.lambda_max(prob), norm_aware=True)
    cc = geo.safe_cc if test == "safe" else geo.dst3_cc
    return (1.0 - np.abs(cc)) / geo.norms
