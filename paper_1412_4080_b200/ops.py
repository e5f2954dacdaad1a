"""Per-op entry points of the hot path, each executed by a libdynscreen kernel.

These mirror the reference's per-op functions (cited below) for callers that
use them directly; the solver engine fuses the same arithmetic into its
per-iteration kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .problem import LambdaMax


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
