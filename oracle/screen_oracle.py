"""CPU oracle for the dynamic-screening solver hot path.

TEST INFRASTRUCTURE ONLY.  This module restates, in numpy, the algorithm of
the reference package ``screenlab`` (``/root/reference/pkg/src/screenlab``) so
that the GPU engine in ``paper_1412_4080_b200`` can be checked against it on
machines where the reference is not installed.  It is imported only by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (the ``cpu_baseline``
leg and ``--impl reference``) -- never by the product package, which fails
loudly when its CUDA library is missing.

Parity is pinned: ``tests/golden/make_golden.py`` runs the reference itself (in
the build container) and commits its outputs under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this restatement against them.

The numerical operations mirror the reference's own numpy calls (reduced
column-major matrices, ``D @ x`` / ``D.T @ v`` GEMVs, the same elementwise
evaluation order) so that on one machine the oracle reproduces the reference
bit for bit.  Each function cites the reference file:line it restates.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

LASSO, GROUP = "lasso", "group"
ISTA, FISTA, TWIST, SPARSA, CP = "ista", "fista", "twist", "sparsa", "cp"
ALGORITHMS = (ISTA, FISTA, TWIST, SPARSA, CP)
NONE, STATIC, DYNAMIC = "none", "static", "dynamic"
SAFE, DST3, DOME, GSAFE, GST3 = "safe", "dst3", "dome", "gsafe", "gst3"
LASSO_TESTS, GROUP_TESTS = (SAFE, DST3, DOME), (GSAFE, GST3)

SCREEN_MARGIN = 1e-12          # screening.py:40
RADIUS_GUARD = 1e-8            # screening.py:33
MAJORIZATION_SLACK = 1e-12     # solvers.py:39
L_CEILING = 1e300              # solvers.py:40
SUPPORT_EPS = 1e-9             # oracle.py:18


# ---------------------------------------------------------------------------
# problem container and group bookkeeping
# ---------------------------------------------------------------------------


@dataclass
class OProblem:
    """Restates problems.Problem (problems.py:20-57) + GroupPartition (dictionary.py:175-216)."""

    D: np.ndarray
    y: np.ndarray
    lam: float
    groups: list | None = None
    weights: np.ndarray | None = None
    snorms: np.ndarray | None = None

    @property
    def kind(self):
        return LASSO if self.groups is None else GROUP

    @property
    def n(self):
        return self.D.shape[0]

    @property
    def k(self):
        return self.D.shape[1]


def make_problem(D, y, lam, groups=None, weights=None, snorms=None):
    D = np.asfortranarray(np.asarray(D, dtype=np.float64))
    y = np.asarray(y, dtype=np.float64)
    if groups is not None:
        groups = [np.asarray(g, dtype=np.int64) for g in groups]
        if weights is None:
            weights = np.sqrt([g.size for g in groups])              # dictionary.py:204-205
        weights = np.asarray(weights, dtype=np.float64)
        if snorms is None:
            snorms = np.array([np.sqrt(power_top_eig(D[:, g])) for g in groups])  # dictionary.py:209
    return OProblem(D, y, float(lam), groups, weights, snorms)


class Layout:
    """Surviving groups inside a reduced coefficient vector (dictionary.py:237-301)."""

    def __init__(self, prob, kept):
        gof = np.empty(prob.k, dtype=np.int64)
        for gid, g in enumerate(prob.groups):
            gof[g] = gid
        self.gids = np.unique(gof[kept]) if kept.size else np.empty(0, np.int64)
        parts = [np.searchsorted(kept, prob.groups[g]) for g in self.gids]
        sizes = np.array([p.size for p in parts], dtype=np.int64)
        self.offsets = (np.concatenate(([0], np.cumsum(sizes)[:-1])) if sizes.size
                        else np.zeros(0, np.int64))
        self.order = np.concatenate(parts) if parts else np.zeros(0, np.int64)
        self.sizes = sizes
        self.weights = prob.weights[self.gids]

    def norms(self, vec):
        if self.order.size == 0:
            return np.zeros(0)
        return np.sqrt(np.add.reduceat(np.asarray(vec)[self.order] ** 2, self.offsets))

    def penalty(self, vec):
        return float(self.weights @ self.norms(vec))

    def shrink(self, vec, t):
        """Group soft threshold with per-group threshold t*w (dictionary.py:290-301)."""
        if t < 0:
            raise ValueError("threshold must be nonnegative")
        nrm = self.norms(vec)
        safe = np.where(nrm > 0.0, nrm, 1.0)
        fac = np.where(nrm > 0.0, np.maximum(1.0 - t * self.weights / safe, 0.0), 0.0)
        out = np.zeros_like(vec)
        out[self.order] = vec[self.order] * np.repeat(fac, self.sizes)
        return out


def full_group_norms(prob, vec):
    """GroupPartition.group_norms over the full index set (dictionary.py:229-235)."""
    order = np.concatenate(prob.groups)
    offs = np.concatenate(([0], np.cumsum([g.size for g in prob.groups])[:-1]))
    return np.sqrt(np.add.reduceat(np.asarray(vec)[order] ** 2, offs))


# ---------------------------------------------------------------------------
# numerical core
# ---------------------------------------------------------------------------


def soft(v, t):
    """Soft threshold sign(v)*max(|v|-t, 0) (problems.py:106-111)."""
    if t < 0:
        raise ValueError("threshold must be nonnegative")
    return np.sign(v) * np.maximum(np.abs(v) - t, 0.0)


@dataclass
class LMax:
    value: float
    index: int | None = None
    atom: np.ndarray | None = None
    group: int | None = None


def lambda_max(prob):
    """Trivial threshold with lowest-index argmax and signed atom (problems.py:75-86)."""
    corr = prob.D.T @ prob.y
    if prob.kind == LASSO:
        i = int(np.argmax(np.abs(corr)))
        sgn = 1.0 if corr[i] >= 0 else -1.0
        return LMax(float(abs(corr[i])), i, sgn * prob.D[:, i])
    ratios = full_group_norms(prob, corr) / prob.weights
    g = int(np.argmax(ratios))
    return LMax(float(ratios[g]), group=g)


def power_top_eig(mat, tol=1e-10, max_iters=5000):
    """Top eigenvalue of mat^T mat by 2-vector block power iteration (dictionary.py:120-158)."""
    rows, cols = mat.shape
    if cols <= rows:
        dim, op = cols, (lambda q: mat.T @ (mat @ q))
    else:
        dim, op = rows, (lambda q: mat @ (mat.T @ q))
    start = [np.ones(dim)]
    if dim > 1:
        alt = np.ones(dim)
        alt[1::2] = -1.0
        start.append(alt)
    q = np.linalg.qr(np.stack(start, axis=1))[0]
    val = None
    for it in range(max_iters):
        z = op(q)
        h = q.T @ z
        new = float(np.linalg.eigvalsh(0.5 * (h + h.T))[-1])
        if val is not None and abs(new - val) <= tol * max(1.0, abs(new)):
            return max(new, 0.0)
        val = new
        if not np.any(z):
            q = np.zeros((dim, q.shape[1]))
            for j in range(q.shape[1]):
                q[(it + j) % dim, j] = 1.0
            val = None
            continue
        q = np.linalg.qr(z)[0]
    return max(val, 0.0)


def operator_norm(D):
    return float(np.sqrt(power_top_eig(D)))


def objective(prob, x):
    """Full objective (problems.py:97-103)."""
    r = prob.D @ x - prob.y
    pen = float(np.sum(np.abs(x))) if prob.kind == LASSO else float(prob.weights @ full_group_norms(prob, x))
    return 0.5 * float(r @ r) + prob.lam * pen


def expand(xr, kept, k):
    out = np.zeros(k)
    out[kept] = xr
    return out


# ---------------------------------------------------------------------------
# screening
# ---------------------------------------------------------------------------


def clip_scale(prob, theta, bound):
    """mu = clip(theta.y / (lam ||theta||^2), +-bound) (screening.py:115-123)."""
    sq = float(theta @ theta)
    if sq == 0.0:
        return 0.0, np.zeros_like(prob.y)
    mu = float(np.clip(float(theta @ prob.y) / (prob.lam * sq), -bound, bound))
    return mu, mu * theta


def dual_scale_lasso(prob, theta, corr_inf=None):
    """screening.py:126-140."""
    if corr_inf is None:
        corr_inf = float(np.max(np.abs(prob.D.T @ theta), initial=0.0))
    return clip_scale(prob, theta, np.inf if corr_inf == 0.0 else 1.0 / corr_inf)


def dual_scale_group(prob, theta, norms=None, weights=None):
    """screening.py:143-165."""
    if norms is None:
        norms = full_group_norms(prob, prob.D.T @ theta)
        weights = prob.weights
    if weights is None:
        weights = prob.weights
    act = norms > 0.0
    bound = float(np.min(weights[act] / norms[act])) if act.any() else np.inf
    return clip_scale(prob, theta, bound)


class Geometry:
    """Per-solve precomputed correlations (ScreeningContext, screening.py:168-322)."""

    def __init__(self, prob, lmax, norm_aware=False):
        self.p, self.lmax = prob, lmax
        self.y_corr = prob.D.T @ prob.y
        self.safe_cc = self.y_corr / prob.lam
        self._cache = {}
        # Extension for reduced-precision dictionaries whose columns are not unit-norm:
        # the sphere test uses ||a_i|| and the DST3 normal is a_*/||a_*||.  At unit norms
        # it reduces to the reference formulas (screening.py:221-231, 351-359).
        self.norms = np.linalg.norm(prob.D, axis=0) if norm_aware else None

    @property
    def star_corr(self):
        if "star" not in self._cache:
            self._cache["star"] = self.p.D.T @ self.lmax.atom
        return self._cache["star"]

    @property
    def shift(self):
        return self.lmax.value / self.p.lam - 1.0

    @property
    def star_norm_sq(self):
        return 1.0 if self.norms is None else float(self.norms[self.lmax.index]) ** 2

    @property
    def dst3_cc(self):
        if self.norms is not None:
            return self.safe_cc - (self.shift / self.star_norm_sq) * self.star_corr
        return self.safe_cc - self.shift * self.star_corr

    def gst3(self):
        if "gst3" not in self._cache:
            p = self.p
            g = self.lmax.group
            sub = p.D[:, p.groups[g]]
            normal = sub @ (sub.T @ p.y) / self.lmax.value
            nsq = float(normal @ normal)
            if nsq == 0.0:
                raise RuntimeError("degenerate extremal group: zero tangent normal")
            coef = float(normal @ p.y) / p.lam - float(p.weights[g]) ** 2
            cc = self.safe_cc - (coef / nsq) * (p.D.T @ normal)
            self._cache["gst3"] = (cc, coef * coef / nsq)
        return self._cache["gst3"]

    def center_group_norms(self, kind):
        key = "norms_" + kind
        if key not in self._cache:
            cc = self.safe_cc if kind == GSAFE else self.gst3()[0]
            self._cache[key] = full_group_norms(self.p, cc)
        return self._cache[key]

    def safe_radius_sq(self, theta, corr_inf=None, norms=None, weights=None):
        if self.p.kind == LASSO:
            mu, v = dual_scale_lasso(self.p, theta, corr_inf)
        else:
            mu, v = dual_scale_group(self.p, theta, norms, weights)
        diff = self.p.y / self.p.lam - v
        return float(diff @ diff), mu

    @staticmethod
    def shifted(rsq, shift_sq):
        arg = rsq - shift_sq
        if arg < -RADIUS_GUARD:
            raise RuntimeError(f"squared screening radius fell to {arg!r}")
        return float(np.sqrt(max(arg, 0.0)))

    def radius(self, kind, theta, corr_inf=None, norms=None, weights=None):
        """Test radius and r_SAFE^2 of a region (screening.py:259-307)."""
        if kind in (DST3, DOME, GST3) and self.p.lam > self.lmax.value:
            raise ValueError("penalty exceeds the trivial-solution threshold")
        rsq, _ = self.safe_radius_sq(theta, corr_inf, norms, weights)
        if kind in (SAFE, GSAFE):
            return float(np.sqrt(rsq)), rsq
        if kind in (DST3, DOME):
            return self.shifted(rsq, self.shift ** 2 / self.star_norm_sq), rsq
        return self.shifted(rsq, self.gst3()[1]), rsq

    def mask(self, kind, r, kept, kept_groups=None):
        if kind in (SAFE, DST3) and self.norms is not None:
            cc = self.safe_cc if kind == SAFE else self.dst3_cc
            return (1.0 - np.abs(cc[kept])) / self.norms[kept] - r > SCREEN_MARGIN
        if kind == SAFE:
            return sphere_mask(self.safe_cc[kept], r)
        if kind == DST3:
            return sphere_mask(self.dst3_cc[kept], r)
        if kind == DOME:
            return dome_mask(self.p.lam, self.lmax.value, self.star_corr[kept], self.y_corr[kept], r)
        gm = group_mask(self.p, kept_groups, self.center_group_norms(kind), r)
        gof = np.empty(self.p.k, dtype=np.int64)
        for gid, g in enumerate(self.p.groups):
            gof[g] = gid
        return gm[np.searchsorted(kept_groups, gof[kept])], gm


def sphere_mask(cc, r):
    """(1 - |cc|) - r > margin (screening.py:351-359)."""
    return (1.0 - np.abs(cc)) - r > SCREEN_MARGIN


def dome_mask(lam, lstar, t, u, radius):
    """Dome test (screening.py:362-388)."""
    if radius >= 1.0:
        return np.zeros(t.size, dtype=bool)
    shift = lstar / lam - 1.0
    rs = float(np.hypot(radius, shift))
    cut = shift / rs if rs > 0.0 else 0.0
    arc = lam * radius * np.sqrt(np.maximum(1.0 - t * t, 0.0))
    slope = lstar - lam
    flat = lam * (1.0 - rs)
    lower = np.where(t < cut, slope * t - lam + arc, -flat)
    upper = np.where(t <= -cut, flat, slope * t + lam - arc)
    m = lam * SCREEN_MARGIN
    return (u - lower > m) & (upper - u > m)


def group_mask(prob, kept_groups, center_norms, r):
    """(w_g - ||D_g^T c||)/||D_g|| - r > margin (screening.py:391-404)."""
    w = prob.weights[kept_groups]
    c = np.asarray(center_norms)[kept_groups]
    s = prob.snorms[kept_groups]
    return (w - c) / s - r > SCREEN_MARGIN


# ---------------------------------------------------------------------------
# solver loop (solvers.py:168-517)
# ---------------------------------------------------------------------------


@dataclass
class Config:
    """Fields of solvers.SolverConfig (solvers.py:44-63) + BASELINE gap stop."""

    algorithm: str = ISTA
    strategy: str = NONE
    test: str | None = None
    max_iters: int = 200
    rel_tol: float = 1e-7
    L0: float = 1.0
    backtrack_factor: float = 2.0
    twist_alpha: float = 1.78
    twist_beta: float = 1.78
    twist_step: float | None = None
    cp_gamma: float = 0.0
    cp_step_safety: float = 0.99
    bb_L_min: float = 1e-10
    bb_L_max: float = 1e10
    gap_tol: float | None = None
    op_norm: float | None = None     # ||D|| override for CP/TwIST (else power iteration)
    norm_aware: bool = False         # non-unit-norm (fp32/bf16-rounded) dictionaries


@dataclass
class OResult:
    x_star: np.ndarray
    iterations: int
    kept: np.ndarray
    eliminated: np.ndarray
    final_objective: float
    trace: dict = field(default_factory=dict)


def flops_iteration(kind, strategy, k, n, kept, nnz, groups=0):
    """Analytic flop model (instrument.py:21-49)."""
    if strategy == NONE:
        kept = k
    base = (kept + nnz) * n
    if strategy in (NONE, STATIC):
        tot = base + 4 * kept + n + (3 * groups if kind == GROUP else 0)
    elif kind == LASSO:
        tot = base + 6 * kept + 5 * n
    else:
        tot = base + 7 * kept + 5 * n + 5 * groups
    return tot


def solve(prob, cfg, hook=None, ticks=None):
    """Restatement of solvers.run (solvers.py:358-511) with an optional gap stop.

    ``ticks`` (a list, optional): ``time.perf_counter()`` is appended once when the iteration
    loop starts (after lambda_max, the screening precomputes and any static screen) and once
    at the end of every iteration -- the CPU baseline times setup and iterations separately.

    The duality gap is the BASELINE quantity F(x_t) - 1/2||y||^2 + lam^2/2 r_SAFE,t^2
    evaluated with the dual point the iteration produced (problems.py:143-149).
    """
    k, n = prob.k, prob.n
    y, lam = prob.y, prob.lam
    group = prob.kind == GROUP
    lm = lambda_max(prob)
    tr = {"t": [], "kept": [], "nnz": [], "objective": [], "gap": [], "radius": [], "flops": []}
    if lam > lm.value:
        return OResult(np.zeros(k), 0, np.empty(0, np.int64), np.arange(k, dtype=np.int64),
                       0.5 * float(y @ y), tr)

    kept = np.arange(k, dtype=np.int64)
    elim = np.empty(0, np.int64)
    geo = Geometry(prob, lm, cfg.norm_aware)
    D = prob.D
    lay = Layout(prob, kept) if group else None
    kept_groups = np.arange(len(prob.groups), dtype=np.int64) if group else None
    flops = 0
    algo = cfg.algorithm

    def prox(v, t):
        return lay.shrink(v, t) if group else soft(v, t)

    def penalty(v):
        return lay.penalty(v) if group else float(np.sum(np.abs(v)))

    if cfg.strategy == STATIC:
        if group:
            norms = full_group_norms(prob, geo.y_corr)
            r, _ = geo.radius(cfg.test, y, norms=norms)
        else:
            r, _ = geo.radius(cfg.test, y, corr_inf=float(np.max(np.abs(geo.y_corr))))
        if group:
            mask, gm = geo.mask(cfg.test, r, kept, kept_groups)
            kept_groups = kept_groups[~gm]
        else:
            mask = geo.mask(cfg.test, r, kept)
        if mask.any():
            elim = np.union1d(elim, kept[mask])
            kept = kept[~mask]
        D = np.asfortranarray(prob.D[:, kept])
        if group:
            lay = Layout(prob, kept)
        flops += k * n

    x = np.zeros(kept.size)
    x_prev = u = theta = corr = resid = None
    L, l_acc, tau, sigma, step = cfg.L0, 1.0, 0.0, 0.0, None
    if algo in (FISTA, CP):
        u = x
    if algo in (CP, TWIST):
        nrm = cfg.op_norm if cfg.op_norm is not None else operator_norm(prob.D)
        if algo == CP:
            tau = sigma = cfg.cp_step_safety / nrm
            theta = np.zeros(n)
        else:
            step = float(cfg.twist_step) if cfg.twist_step is not None else 1.0 / nrm ** 2

    def backtrack(point, th, c, L):
        f0 = 0.5 * float(th @ th)
        while True:
            cand = prox(point - c / L, lam / L)
            rc = D @ cand - y
            fc = 0.5 * float(rc @ rc)
            d = cand - point
            bound = f0 + float(c @ d) + 0.5 * L * float(d @ d)
            if fc <= bound + MAJORIZATION_SLACK * max(1.0, f0):
                return cand, rc, L
            L *= cfg.backtrack_factor
            if L > L_CEILING:
                raise FloatingPointError("backtracking failed to find a valid step")

    def finite(v):
        if not np.all(np.isfinite(v)):
            raise FloatingPointError("solver produced a non-finite iterate")

    f_prev, moved, it = None, False, 0
    if ticks is not None:
        ticks.append(time.perf_counter())
    for t in range(1, cfg.max_iters + 1):
        if kept.size == 0:
            break
        # -- update (solvers.py:190-313)
        if algo == ISTA:
            theta = resid if resid is not None else D @ x - y
            corr = D.T @ theta
            cand, rc, L = backtrack(x, theta, corr, L)
            finite(cand)
            x_prev, x, resid = x, cand, rc
        elif algo == FISTA:
            pt = u if u is not None else x
            theta = D @ pt - y
            corr = D.T @ theta
            cand, rc, L = backtrack(pt, theta, corr, L)
            finite(cand)
            l_new = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * l_acc ** 2))
            u = cand + ((l_acc - 1.0) / l_new) * (cand - x)
            l_acc = float(l_new)
            x_prev, x, resid = x, cand, rc
        elif algo == SPARSA:
            theta = resid if resid is not None else D @ x - y
            corr = D.T @ theta
            if x_prev is not None:
                s = x - x_prev
                ss = float(s @ s)
                if ss > 0.0:
                    ds = D @ s
                    L = float(np.clip(float(ds @ ds) / ss, cfg.bb_L_min, cfg.bb_L_max))
            cand = prox(x - corr / L, lam / L)
            finite(cand)
            x_prev, x, resid = x, cand, None
        elif algo == CP:
            pt = u if u is not None else x
            th_prev = theta if theta is not None else np.zeros_like(y)
            theta = (th_prev + sigma * (D @ pt - y)) / (1.0 + sigma)
            corr = D.T @ theta
            cand = prox(x - tau * corr, lam * tau)
            finite(cand)
            phi = 1.0 / np.sqrt(1.0 + 2.0 * cfg.cp_gamma * tau)
            u = cand + phi * (cand - x)
            tau, sigma = float(phi * tau), float(sigma / phi)
            x_prev, x, resid = x, cand, None
        else:  # TWIST
            theta = resid if resid is not None else D @ x - y
            corr = D.T @ theta
            z = prox(x - step * corr, lam * step)
            if x_prev is None:
                cand = z
            else:
                a, b = cfg.twist_alpha, cfg.twist_beta
                cand = (1.0 - a) * x_prev + (a - b) * x + b * z
            finite(cand)
            x_prev, x, resid = x, cand, None
        it = t

        # -- dual scaling at theta_t over the pre-screening set; dynamic test
        if group:
            gnorms = lay.norms(corr)
            rsafe_sq, _ = geo.safe_radius_sq(theta, norms=gnorms, weights=lay.weights)
        else:
            cinf = float(np.max(np.abs(corr), initial=0.0))
            rsafe_sq, _ = geo.safe_radius_sq(theta, corr_inf=cinf)
        mask, radius = None, float("nan")
        if cfg.strategy == DYNAMIC:
            if group:
                radius, _ = geo.radius(cfg.test, theta, norms=gnorms, weights=lay.weights)
                mask, _ = geo.mask(cfg.test, radius, kept, kept_groups)
            else:
                radius, _ = geo.radius(cfg.test, theta, corr_inf=cinf)
                mask = geo.mask(cfg.test, radius, kept)
        if hook is not None:
            hook({"t": t, "theta": theta, "corr": corr, "kept": kept, "kept_groups": kept_groups,
                  "mask": mask, "x": x, "radius": radius, "rsafe_sq": rsafe_sq})
        if mask is not None and mask.any():
            keep = np.flatnonzero(~mask)
            dropped_zero = bool(np.all(x[mask] == 0.0))
            elim = np.union1d(elim, kept[mask])
            kept = kept[~mask]
            if keep.size != D.shape[1]:
                D = np.asfortranarray(D[:, keep])
            if group:
                lay = Layout(prob, kept)
                kept_groups = lay.gids
            x = x[keep]
            if x_prev is not None:
                x_prev = x_prev[keep]
            if u is not None:
                u = u[keep]
            corr = None
            if not dropped_zero:
                resid = None
        if resid is None:
            resid = D @ x - y
        f_t = 0.5 * float(resid @ resid) + lam * penalty(x)
        nnz = int(np.count_nonzero(x))
        flops += flops_iteration(prob.kind, cfg.strategy, k, n, kept.size, nnz,
                                 len(prob.groups) if group else 0)
        gap = f_t - 0.5 * float(y @ y) + 0.5 * lam * lam * rsafe_sq
        for key, val in (("t", t), ("kept", kept.size), ("nnz", nnz), ("objective", f_t),
                         ("gap", gap), ("radius", radius), ("flops", flops)):
            tr[key].append(val)
        if ticks is not None:
            ticks.append(time.perf_counter())
        moved = moved or nnz > 0
        if moved and f_prev is not None and abs(f_prev - f_t) / max(f_t, 1e-300) < cfg.rel_tol:
            break
        if cfg.gap_tol is not None and gap <= cfg.gap_tol:
            break
        f_prev = f_t

    final = tr["objective"][-1] if tr["objective"] else 0.5 * float(y @ y)
    return OResult(expand(x, kept, k), it, kept, elim, final, tr)


# ---------------------------------------------------------------------------
# certified coordinate-descent reference (oracle.py:34-139)
# ---------------------------------------------------------------------------


def certified_gap(prob, x, resid):
    theta = resid / prob.lam
    if prob.kind == LASSO:
        _, v = dual_scale_lasso(prob, theta)
        feas = float(np.max(np.abs(prob.D.T @ v), initial=0.0)) <= 1.0 + 1e-12
    else:
        _, v = dual_scale_group(prob, theta)
        feas = bool(np.all(full_group_norms(prob, prob.D.T @ v) <= prob.weights * (1.0 + 1e-12)))
    if not feas:
        raise ValueError("theta is not dual feasible")
    primal = objective(prob, x)
    diff = v - prob.y / prob.lam
    gap = primal - (0.5 * float(prob.y @ prob.y) - 0.5 * prob.lam ** 2 * float(diff @ diff))
    if gap < 0.0:
        if gap < -1e-12 * max(1.0, abs(primal)):
            raise ValueError("negative duality gap")
        gap = 0.0
    return gap


def cd_solve(prob, gap_tol=1e-10, max_sweeps=200_000):
    """Cyclic (block) coordinate descent to a certified gap (oracle.py:44-125)."""
    lm = lambda_max(prob)
    k = prob.k
    if prob.lam > lm.value:
        return np.zeros(k), certified_gap(prob, np.zeros(k), prob.y.copy())
    d, lam = prob.D, prob.lam
    x = np.zeros(k)
    res = prob.y.copy()
    if prob.kind == LASSO:
        csq = np.einsum("ij,ij->j", d, d)

        def sweep(ids):
            mv = 0.0
            for i in ids:
                xi = x[i]
                rho = float(d[:, i] @ res) + csq[i] * xi
                xn = np.sign(rho) * max(abs(rho) - lam, 0.0) / csq[i]
                if xn != xi:
                    res[:] += d[:, i] * (xi - xn)
                    x[i] = xn
                    mv = max(mv, abs(xn - xi))
            return mv

        def support():
            return np.flatnonzero(x != 0.0)
    else:
        lip = np.maximum(prob.snorms ** 2, 1e-300)

        def sweep(ids):
            mv = 0.0
            for g in ids:
                idx = prob.groups[g]
                sub = d[:, idx]
                xg = x[idx]
                z = xg + (sub.T @ res) / lip[g]
                nz = float(np.linalg.norm(z))
                thr = lam * prob.weights[g] / lip[g]
                xn = z * max(1.0 - thr / nz, 0.0) if nz > 0.0 else np.zeros_like(z)
                delta = xn - xg
                if np.any(delta != 0.0):
                    res[:] -= sub @ delta
                    x[idx] = xn
                    mv = max(mv, float(np.max(np.abs(delta))))
            return mv

        def support():
            return np.flatnonzero(full_group_norms(prob, x) != 0.0)

    units = np.arange(k if prob.kind == LASSO else len(prob.groups))
    sweeps = 0
    while sweeps < max_sweeps:
        sweep(units)
        sweeps += 1
        gap = certified_gap(prob, x, res)
        if gap <= gap_tol:
            return x.copy(), gap
        ids = support()
        for _ in range(10):
            if ids.size == 0 or sweeps >= max_sweeps:
                break
            mv = sweep(ids)
            sweeps += 1
            if mv < 1e-16:
                break
    raise RuntimeError(f"reference solver hit {max_sweeps} sweeps before gap <= {gap_tol!r}")


def screen_is_safe(x_ref, eliminated, eps=SUPPORT_EPS):
    """verify_screen_safety (oracle.py:128-139)."""
    eliminated = np.asarray(eliminated, dtype=np.int64)
    return bool(eliminated.size == 0 or np.all(np.abs(x_ref[eliminated]) <= eps))
