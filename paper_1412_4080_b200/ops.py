"""Per-op entry points of the hot path, each executed by a libdynscreen kernel.

These mirror the reference's per-op functions (cited below) for callers that
use them directly; the solver engine fuses the same arithmetic into its
per-iteration kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .problem import LambdaMax, index_set


def _dev():
    import torch
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, dtype=None):
    import torch
    t = torch.from_numpy(np.array(a, copy=True, order="C"))
    return t.to(_dev()) if dtype is None else t.to(_dev(), dtype)


@dataclass(frozen=True)
class SphereRegion:
    """screening.py:46-55."""

    center: np.ndarray
    radius: float
    center_correlations: np.ndarray


@dataclass(frozen=True)
class DomeParams:
    """screening.py:59-80."""

    lam: float
    lambda_star: float
    star_correlations: np.ndarray
    y_correlations: np.ndarray
    radius: float

    def __post_init__(self):
        for name in ("star_correlations", "y_correlations"):
            arr = np.asarray(getattr(self, name))
            if arr.size and float(np.max(np.abs(arr))) > 1.0 + 1e-9:
                raise ValueError(f"{name} must lie in [-1, 1] up to roundoff")


def prox_l1(x, t):
    """Soft thresholding on the device (problems.py:106-111)."""
    import torch
    if t < 0:
        raise ValueError("threshold must be nonnegative")
    x = np.asarray(x, dtype=np.float64)
    L = nat.lib()
    xd = _to_dev(x.ravel())
    out = torch.empty_like(xd)
    nat.check(L.dscr_prox_l1(xd.data_ptr(), xd.numel(), float(t), out.data_ptr(), nat.stream_ptr()))
    return out.cpu().numpy().reshape(x.shape)


def prox_group(x, t, partition):
    """Group soft thresholding with per-group threshold t*w_g (problems.py:114-125)."""
    import torch
    if t < 0:
        raise ValueError("threshold must be nonnegative")
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (partition.size,):
        raise ValueError(f"expected coefficient vector of length {partition.size}")
    order = np.concatenate(partition.groups)
    ptr = np.concatenate(([0], np.cumsum(partition.group_sizes()))).astype(np.int32)
    L = nat.lib()
    vd, pd = _to_dev(x[order]), _to_dev(ptr)
    wd = _to_dev(np.asarray(partition.weights, np.float64))
    out = torch.empty_like(vd)
    nat.check(L.dscr_prox_group(vd.data_ptr(), pd.data_ptr(), partition.n_groups, wd.data_ptr(), float(t),
                                out.data_ptr(), nat.stream_ptr()))
    res = np.zeros_like(x)
    res[order] = out.cpu().numpy()
    return res


def lambda_max(problem):
    """Trivial threshold and extremal atom/group (problems.py:75-86); correlations on the device."""
    corr = problem.dictionary.correlate(problem.y)
    if problem.kind == "lasso":
        i = int(np.argmax(np.abs(corr)))
        sign = 1.0 if corr[i] >= 0 else -1.0
        return LambdaMax(float(abs(corr[i])), sign * problem.dictionary.column(i), i)
    part = problem.partition
    norms = np.array([np.sqrt(np.sum(corr[g] ** 2)) for g in part.groups])
    ratios = norms / part.weights
    g = int(np.argmax(ratios))
    return LambdaMax(float(ratios[g]), group=g)


def test_sphere_lasso(region, kept):
    """(1 - |c_i|) - r > 1e-12 over `kept` (screening.py:351-359)."""
    import torch
    kept = np.asarray(kept, dtype=np.int32)
    L = nat.lib()
    cc = _to_dev(np.asarray(region.center_correlations, np.float64))
    kd = _to_dev(kept)
    out = torch.empty(max(kept.size, 1), dtype=torch.uint8, device=_dev())
    nat.check(L.dscr_test_sphere(cc.data_ptr(), kd.data_ptr(), kept.size, float(region.radius), out.data_ptr(),
                                 nat.stream_ptr()))
    return out[: kept.size].cpu().numpy().astype(bool)


def test_dome(dp, kept):
    """Dome test (screening.py:362-388)."""
    import torch
    kept = np.asarray(kept, dtype=np.int32)
    L = nat.lib()
    out = torch.empty(max(kept.size, 1), dtype=torch.uint8, device=_dev())
    td = _to_dev(np.asarray(dp.star_correlations, np.float64))
    ud = _to_dev(np.asarray(dp.y_correlations, np.float64))
    kd = _to_dev(kept)
    nat.check(L.dscr_test_dome(td.data_ptr(), ud.data_ptr(), kd.data_ptr(), kept.size, float(dp.lam),
                               float(dp.lambda_star), float(dp.radius), out.data_ptr(), nat.stream_ptr()))
    return out[: kept.size].cpu().numpy().astype(bool)


def test_sphere_group(region, partition, kept_groups, center_group_norms=None):
    """(w_g - ||D_g^T c||)/||D_g|| - r > 1e-12 (screening.py:391-404)."""
    import torch
    kept_groups = np.asarray(kept_groups, dtype=np.int32)
    if center_group_norms is None:
        cc = np.asarray(region.center_correlations, np.float64)
        center_group_norms = np.array([np.sqrt(np.sum(cc[g] ** 2)) for g in partition.groups])
    L = nat.lib()
    out = torch.empty(max(kept_groups.size, 1), dtype=torch.uint8, device=_dev())
    wd = _to_dev(np.asarray(partition.weights, np.float64))
    cd = _to_dev(np.asarray(center_group_norms, np.float64))
    sd = _to_dev(np.asarray(partition.spectral_norms, np.float64))
    kd = _to_dev(kept_groups)
    nat.check(L.dscr_test_group(wd.data_ptr(), cd.data_ptr(), sd.data_ptr(), kd.data_ptr(), kept_groups.size,
                                float(region.radius), out.data_ptr(), nat.stream_ptr()))
    return out[: kept_groups.size].cpu().numpy().astype(bool)


def screen_update(state, mask):
    """Fold an elimination mask aligned with ``state.kept`` (screening.py:104-112).

    Host set algebra on the ScreenState container; the engine itself compacts
    its active list on the device."""
    from .solver import ScreenState
    mask = np.asarray(mask, dtype=bool)
    if mask.shape != (state.kept.size,):
        raise ValueError("mask must align with the kept index set")
    if not mask.any():
        return state
    eliminated = np.union1d(state.eliminated, state.kept[mask])
    return ScreenState(eliminated=eliminated, kept=state.kept[~mask], test_kind=state.test_kind)


# ---- inner seams of the iteration (kernel-level entry points) -----------------


def _theta_dev(dictionary, theta):
    import torch
    theta = np.asarray(theta, dtype=np.float64)
    if theta.shape != (dictionary.n_rows,):
        raise ValueError(f"expected observation-space vector of length {dictionary.n_rows}")
    out = torch.zeros(dictionary.ldd, dtype=torch.float64, device=_dev())
    out[: dictionary.n_rows].copy_(torch.from_numpy(theta))
    return out


def _coef_dev(dictionary, v, name):
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (dictionary.n_cols,):
        raise ValueError(f"{name} must have one entry per atom ({dictionary.n_cols})")
    return _to_dev(v)


def _step_args(L=None, tau=None):
    if (L is None) == (tau is None):
        raise ValueError("give exactly one of L (v = point - c/L) or tau (v = point - tau*c)")
    return (float(L), 0) if L is not None else (float(tau), 1)


def corr_prox(dictionary, active, theta, point, lam, L=None, tau=None, x_prev=None, beta=0.0):
    """One proximal gradient step over the active atoms on the device (update_ista /
    update_fista's step, solvers.py:168-225): ``corr = D_A^T theta``, ``x = prox_l1(point -
    corr/L, lam/L)`` (or ``point - tau*corr`` with threshold ``lam*tau``: CP / TwIST), and with
    ``x_prev`` the FISTA point ``u = x + beta (x - x_prev)``.  Coefficient vectors are full
    length (one entry per atom); atoms outside ``active`` are returned unchanged (zero).
    Returns ``(x, u or None, corr, (max|corr|, corr.(x - point), ||x - point||^2))``."""
    import torch
    active = index_set(active, dictionary.n_cols)
    s, mult = _step_args(L, tau)
    thr = float(lam) / s if mult == 0 else float(lam) * s
    dev = _dev()
    D = dictionary.device_data(dev)
    th = _theta_dev(dictionary, theta)
    pt = _coef_dev(dictionary, point, "point")
    xp = _coef_dev(dictionary, x_prev, "x_prev") if x_prev is not None else None
    act = _to_dev(active.astype(np.int32))
    x_out = torch.zeros(dictionary.n_cols, dtype=torch.float64, device=dev)
    u_out = torch.zeros_like(x_out) if xp is not None else None
    corr = torch.zeros_like(x_out)
    red = torch.zeros(3, dtype=torch.float64, device=dev)
    L_ = nat.lib()
    nat.check(L_.dscr_corr_prox(dictionary.dtype_code, D.data_ptr(), dictionary.ldd, dictionary.n_rows,
                                act.data_ptr(), int(active.size), th.data_ptr(), pt.data_ptr(),
                                xp.data_ptr() if xp is not None else None, s, mult, thr, float(beta),
                                x_out.data_ptr(), u_out.data_ptr() if u_out is not None else None,
                                corr.data_ptr(), red.data_ptr(), nat.stream_ptr()))
    r = red.cpu().numpy()
    return (x_out.cpu().numpy(), None if u_out is None else u_out.cpu().numpy(), corr.cpu().numpy(),
            (float(r[0]), float(r[1]), float(r[2])))


def group_corr_prox(dictionary, partition, active_groups, theta, point, lam, L=None, tau=None, x_prev=None,
                    beta=0.0):
    """The group-Lasso step on the device (GroupLayout.prox of the gradient step,
    dictionary.py:290-301): correlations of the active groups' atoms, block soft threshold with
    per-group threshold ``(lam/L) w_g``.  The partition's groups must be contiguous column
    ranges in order.  Returns ``(x, u or None, corr, group_corr_norms, (min_g w_g/||c_g||,
    corr.(x - point), ||x - point||^2))``."""
    import torch
    groups = [np.asarray(g, dtype=np.int64) for g in partition.groups]
    order = np.concatenate(groups)
    if not np.array_equal(order, np.arange(dictionary.n_cols)):
        raise ValueError("the seam entry points need contiguous groups in column order")
    active_groups = index_set(active_groups, partition.n_groups)
    ptr = np.concatenate(([0], np.cumsum([g.size for g in groups]))).astype(np.int32)
    atoms = np.concatenate([groups[g] for g in active_groups]) if active_groups.size else np.empty(0, np.int64)
    s, mult = _step_args(L, tau)
    thr = float(lam) / s if mult == 0 else float(lam) * s
    dev = _dev()
    D = dictionary.device_data(dev)
    th = _theta_dev(dictionary, theta)
    pt = _coef_dev(dictionary, point, "point")
    xp = _coef_dev(dictionary, x_prev, "x_prev") if x_prev is not None else None
    gp, ag, aa = _to_dev(ptr), _to_dev(active_groups.astype(np.int32)), _to_dev(atoms.astype(np.int32))
    w = _to_dev(np.asarray(partition.weights, dtype=np.float64))
    x_out = torch.zeros(dictionary.n_cols, dtype=torch.float64, device=dev)
    u_out = torch.zeros_like(x_out) if xp is not None else None
    corr = torch.zeros_like(x_out)
    cn = torch.zeros(max(1, active_groups.size), dtype=torch.float64, device=dev)
    red = torch.zeros(3, dtype=torch.float64, device=dev)
    L_ = nat.lib()
    nat.check(L_.dscr_group_corr_prox(dictionary.dtype_code, D.data_ptr(), dictionary.ldd, dictionary.n_rows,
                                      gp.data_ptr(), ag.data_ptr(), int(active_groups.size), aa.data_ptr(),
                                      int(atoms.size), w.data_ptr(), th.data_ptr(), pt.data_ptr(),
                                      xp.data_ptr() if xp is not None else None, s, mult, thr, float(beta),
                                      x_out.data_ptr(), u_out.data_ptr() if u_out is not None else None,
                                      corr.data_ptr(), cn.data_ptr(), red.data_ptr(), nat.stream_ptr()))
    r = red.cpu().numpy()
    return (x_out.cpu().numpy(), None if u_out is None else u_out.cpu().numpy(), corr.cpu().numpy(),
            cn[: active_groups.size].cpu().numpy(), (float(r[0]), float(r[1]), float(r[2])))


def residual(dictionary, idx, x, y, u=None):
    """``D_S x - y`` (and ``D_S u - y``) over a compact support list on the device
    (solvers.py:160-165, dictionary.py:82-87).  Returns ``(r_x, r_u or None, (||r_x||^2,
    ||r_u||^2, r_u.y))``."""
    import torch
    idx = np.asarray(idx, dtype=np.int64)
    x = np.asarray(x, dtype=np.float64)
    if idx.ndim != 1 or x.shape != idx.shape or (u is not None and np.asarray(u).shape != idx.shape):
        raise ValueError("idx, x (and u) must be aligned 1-D arrays")
    if idx.size and (idx.min() < 0 or idx.max() >= dictionary.n_cols):
        raise ValueError(f"indices must lie in [0, {dictionary.n_cols})")
    y = np.asarray(y, dtype=np.float64)
    if y.shape != (dictionary.n_rows,):
        raise ValueError("observation length must match the dictionary rows")
    dev = _dev()
    D = dictionary.device_data(dev)
    n = dictionary.n_rows
    idd = _to_dev(idx.astype(np.int32)) if idx.size else torch.zeros(1, dtype=torch.int32, device=dev)
    xd = _to_dev(x) if idx.size else torch.zeros(1, dtype=torch.float64, device=dev)
    ud = None
    if u is not None:
        ud = _to_dev(np.asarray(u, dtype=np.float64)) if idx.size else torch.zeros(1, dtype=torch.float64, device=dev)
    yd = _to_dev(y)
    rx = torch.empty(n, dtype=torch.float64, device=dev)
    ru = torch.empty(n, dtype=torch.float64, device=dev) if ud is not None else None
    red = torch.zeros(3, dtype=torch.float64, device=dev)
    nat.check(nat.lib().dscr_residual(dictionary.dtype_code, D.data_ptr(), dictionary.ldd, n, idd.data_ptr(),
                                      int(idx.size), xd.data_ptr(), ud.data_ptr() if ud is not None else None,
                                      yd.data_ptr(), rx.data_ptr(), ru.data_ptr() if ru is not None else None,
                                      red.data_ptr(), nat.stream_ptr()))
    r = red.cpu().numpy()
    return rx.cpu().numpy(), None if ru is None else ru.cpu().numpy(), (float(r[0]), float(r[1]), float(r[2]))


def compact(active, mask):
    """Order-preserving compaction ``active[~mask]`` on the device (the kept set of
    screen_update, screening.py:104-112)."""
    import torch
    active = np.asarray(active, dtype=np.int64)
    mask = np.asarray(mask, dtype=bool)
    if mask.shape != active.shape or active.ndim != 1:
        raise ValueError("mask must align with the active list")
    dev = _dev()
    n = int(active.size)
    a = _to_dev(active.astype(np.int32)) if n else torch.zeros(1, dtype=torch.int32, device=dev)
    m = _to_dev(mask.astype(np.uint8)) if n else torch.zeros(1, dtype=torch.uint8, device=dev)
    out = torch.empty(max(1, n), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    L_ = nat.lib()
    nb = int(L_.dscr_compact_work_size(n))
    work = torch.empty(nb, dtype=torch.uint8, device=dev)
    nat.check(L_.dscr_compact(a.data_ptr(), n, m.data_ptr(), out.data_ptr(), cnt.data_ptr(), work.data_ptr(), nb,
                              nat.stream_ptr()))
    k = int(cnt.item())
    return out[:k].cpu().numpy().astype(np.int64)
