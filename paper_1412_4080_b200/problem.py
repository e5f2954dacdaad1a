"""Host-side problem types mirroring the reference's public containers.

``Dictionary`` (reference dictionary.py:37-117), ``GroupPartition``
(dictionary.py:175-264), ``Problem`` / ``LambdaMax`` (problems.py:20-72).  The
host objects validate exactly like the reference and own the host arrays; the
numerical work (correlations, products, spectral norms, lambda_max) runs on the
GPU through libdynscreen.  Device copies are cached on the object, so a
lambda sweep over one dictionary uploads it once.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat

UNIT_NORM_TOL = 1e-9      # dictionary.py:10
OBS_NORM_TOL = 1e-9       # problems.py:13
LASSO = "lasso"
GROUP = "group"

_DTYPES = {"f64": (np.float64, nat.F64), "f32": (np.float32, nat.F32), "bf16": (np.uint16, nat.BF16)}


def index_set(values, size=None):
    """Strictly increasing int64 index array (dictionary.py:17-27)."""
    arr = np.asarray(values, dtype=np.int64).ravel()
    if arr.size and np.any(np.diff(arr) <= 0):
        raise ValueError("index set must be strictly increasing")
    if size is not None and arr.size and (arr[0] < 0 or arr[-1] >= size):
        raise ValueError(f"indices must lie in [0, {size})")
    return arr


def _pad16(n):
    return (n + 15) // 16 * 16


class Dictionary:
    """Dense N x K column-major dictionary (reference dictionary.py:37-117).

    ``dtype`` selects the device storage: "f64" (the default and the reference's: any input,
    float32 included, is upcast as ``np.array(data, dtype=np.float64)`` does in
    dictionary.py:48), "f32" or "bf16" (bit patterns passed as uint16) on request.  All
    arithmetic accumulates in fp64.  The unit-norm check (tolerance 1e-9) runs on the exact
    fp64 upcast; see ``norm_aware`` for which screening formulas a solve uses.
    """

    def __init__(self, data, check_unit_norms=True, dtype=None):
        if dtype is None:
            dtype = "f64"
        if dtype not in _DTYPES:
            raise ValueError(f"unknown dictionary dtype {dtype!r}")
        np_t, code = _DTYPES[dtype]
        arr = np.asarray(data)
        if arr.dtype != np_t or not arr.flags.f_contiguous:
            arr = np.array(data, dtype=np_t, order="F")
        if arr.ndim != 2:
            raise ValueError("dictionary data must be a 2-D matrix")
        n, k = arr.shape
        if n < 1 or k < 1:
            raise ValueError("dictionary must have at least one row and one column")
        if check_unit_norms:
            worst = 0.0
            for c0 in range(0, k, 8192):
                blk = self._upcast(arr[:, c0:c0 + 8192], dtype)
                worst = max(worst, float(np.max(np.abs(np.linalg.norm(blk, axis=0) - 1.0))))
            if worst > UNIT_NORM_TOL:
                raise ValueError(f"columns must have unit l2 norm (worst deviation {worst:.3e})")
        self.data = arr
        self.dtype = dtype
        self.dtype_code = code
        self.col_norm_checked = bool(check_unit_norms)
        self._dev = {}
        self._op_norm = None

    @property
    def norm_aware(self):
        """Whether the screening tests use the norm-aware generalisation ((1 - |a_i.c|)/||a_i||,
        DST3 normal a*/||a*||) instead of the reference's unit-atom formulas.  fp64 storage always
        follows the reference (which never looks at column norms, checked or not: an fp64
        dictionary built with ``check_unit_norms=False`` gets exactly the reference's tests,
        radius guard included); reduced-precision storage whose rounded columns did not pass the
        1e-9 unit-norm check uses the generalisation, which stays safe at any column norm."""
        return self.dtype != "f64" and not self.col_norm_checked

    @staticmethod
    def _upcast(a, dtype):
        if dtype == "bf16":
            return (np.asarray(a, dtype=np.uint32) << 16).view(np.float32).astype(np.float64)
        return np.asarray(a, dtype=np.float64)

    @property
    def n_rows(self):
        return self.data.shape[0]

    @property
    def n_cols(self):
        return self.data.shape[1]

    @property
    def ldd(self):
        return _pad16(self.n_rows)

    def column(self, i):
        return self._upcast(self.data[:, i], self.dtype)

    def as_float64(self):
        return self._upcast(self.data, self.dtype)

    # -- device residency ------------------------------------------------
    def device_data(self, device, perm=None):
        """Column-major padded device copy (ldd x K), optionally column-permuted."""
        import torch
        key = (str(device), None if perm is None else perm.tobytes())
        hit = self._dev.get(key)
        if hit is not None:
            return hit
        n, k, ldd = self.n_rows, self.n_cols, self.ldd
        pinned = self.__dict__.get("_host_tensor")
        if perm is None and pinned is not None:
            src = pinned                                                 # pinned (K, N) view of self.data
        else:
            host = self.data if perm is None else np.asfortranarray(self.data[:, perm])
            src = torch.from_numpy(np.ascontiguousarray(host.T))       # (K, N) rows = columns
        if ldd == n:
            dev = src.to(device, non_blocking=True)
        else:
            dev = torch.zeros((k, ldd), dtype=src.dtype, device=device)
            dev[:, :n].copy_(src, non_blocking=True)
        self._dev[key] = dev
        return dev

    def drop_device(self):
        """Forget every device copy (the dictionary, the per-partition arrays and column norms
        the solver caches on it): the next solve uploads again."""
        self._dev.clear()
        self.__dict__.pop("_problem_cache", None)

    # -- GPU-backed operators --------------------------------------------
    def apply(self, x):
        """D @ x on the device (dictionary.py:82-87)."""
        import torch
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n_cols,):
            raise ValueError(f"expected coefficient vector of length {self.n_cols}")
        dev = torch.device("cuda", torch.cuda.current_device())
        L = nat.lib()
        Dd = self.device_data(dev)
        xd = torch.from_numpy(x).to(dev)
        out = torch.empty(self.ldd, dtype=torch.float64, device=dev)
        nb = int(L.dscr_apply_work_size(self.dtype_code, self.ldd, self.n_cols))
        work = torch.empty(nb, dtype=torch.uint8, device=dev)
        nat.check(L.dscr_apply(self.dtype_code, Dd.data_ptr(), self.ldd, self.n_rows, self.n_cols,
                               xd.data_ptr(), out.data_ptr(), work.data_ptr(), nb, nat.stream_ptr()))
        return out[: self.n_rows].cpu().numpy()

    def correlate(self, v):
        """D.T @ v on the device (dictionary.py:89-94)."""
        import torch
        v = np.asarray(v, dtype=np.float64)
        if v.shape != (self.n_rows,):
            raise ValueError(f"expected observation-space vector of length {self.n_rows}")
        dev = torch.device("cuda", torch.cuda.current_device())
        L = nat.lib()
        Dd = self.device_data(dev)
        vd = torch.zeros(self.ldd, dtype=torch.float64, device=dev)
        vd[: self.n_rows].copy_(torch.from_numpy(v))
        out = torch.empty(self.n_cols, dtype=torch.float64, device=dev)
        nat.check(L.dscr_correlate(self.dtype_code, Dd.data_ptr(), self.ldd, self.n_rows, self.n_cols,
                                   vd.data_ptr(), out.data_ptr(), nat.stream_ptr()))
        return out.cpu().numpy()

    def reduce(self, kept_prev, kept_next):
        """Sub-dictionary of the kept columns (dictionary.py:99-117)."""
        kept_prev = index_set(kept_prev)
        kept_next = index_set(kept_next)
        if kept_prev.size != self.n_cols:
            raise ValueError("kept_prev does not match the current column count")
        pos = np.searchsorted(kept_prev, kept_next)
        if np.any(pos >= kept_prev.size) or np.any(kept_prev[np.minimum(pos, kept_prev.size - 1)] != kept_next):
            raise ValueError("kept_next must be a subset of kept_prev")
        if kept_next.size == kept_prev.size:
            return self
        out = Dictionary.__new__(Dictionary)
        out.data = np.asfortranarray(self.data[:, pos])
        out.dtype, out.dtype_code = self.dtype, self.dtype_code
        out.col_norm_checked = self.col_norm_checked
        out._dev, out._op_norm = {}, None
        return out


def operator_norm(dictionary, cols=None, tol=1e-10, max_iters=5000):
    """Largest singular value by 2-vector block power iteration on the GPU
    (dictionary.py:120-171)."""
    import torch
    L = nat.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    if cols is None:
        Dd = dictionary.device_data(dev)
        k = dictionary.n_cols
    else:
        cols = index_set(cols, dictionary.n_cols)
        if cols.size == 0:
            raise ValueError("spectral_norm requires a nonempty column set")
        base = dictionary.device_data(dev)
        src = base.view(torch.int16) if base.dtype == torch.uint16 else base    # bf16 bits: gather as int16
        Dd = src[torch.from_numpy(cols).to(dev)].contiguous().view(base.dtype)
        k = int(cols.size)
    ldd = dictionary.ldd
    work = torch.empty(int(L.dscr_operator_norm_work_size(ldd, k)), dtype=torch.uint8, device=dev)
    out = nat.C.c_double(0.0)
    nat.check(L.dscr_operator_norm(dictionary.dtype_code, Dd.data_ptr(), ldd, dictionary.n_rows, k, tol,
                                   max_iters, work.data_ptr(), nat.C.byref(out), nat.stream_ptr()))
    return float(out.value)


def spectral_norm(dictionary, cols):
    return operator_norm(dictionary, cols)


def group_spectral_norms(dictionary, groups, tol=1e-10, max_iters=5000):
    """||D_g||_2 for every group in one kernel (dscr_group_spectral_norms: per-group fp64 Gram
    + the same block power iteration); groups the kernel does not take (> 32 columns or more
    columns than rows) go through operator_norm."""
    import torch
    L = nat.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    groups = [index_set(g, dictionary.n_cols) for g in groups]
    if any(g.size == 0 for g in groups):
        raise ValueError("spectral_norm requires a nonempty column set")
    ptr = np.zeros(len(groups) + 1, dtype=np.int32)
    ptr[1:] = np.cumsum([g.size for g in groups])
    cols = np.concatenate(groups).astype(np.int32)
    Dd = dictionary.device_data(dev)
    ptr_d, cols_d = torch.from_numpy(ptr).to(dev), torch.from_numpy(cols).to(dev)
    out = torch.empty(len(groups), dtype=torch.float64, device=dev)
    nat.check(L.dscr_group_spectral_norms(dictionary.dtype_code, Dd.data_ptr(), dictionary.ldd, dictionary.n_rows,
                                          len(groups), ptr_d.data_ptr(), cols_d.data_ptr(), float(tol),
                                          int(max_iters), out.data_ptr(), nat.stream_ptr()))
    norms = out.cpu().numpy()
    for gi in np.flatnonzero(norms < 0):
        norms[gi] = operator_norm(dictionary, groups[gi], tol=tol, max_iters=max_iters)
    return norms


@dataclass(frozen=True)
class GroupPartition:
    """Weighted partition of the columns (dictionary.py:175-264)."""

    groups: tuple
    weights: np.ndarray
    spectral_norms: np.ndarray
    group_of: np.ndarray
    order: np.ndarray
    offsets: np.ndarray

    @classmethod
    def build(cls, dictionary, groups, weights=None, spectral_norms=None):
        k = dictionary.n_cols
        groups = tuple(index_set(g, k) for g in groups)
        if any(g.size == 0 for g in groups):
            raise ValueError("groups must be nonempty")
        group_of = np.full(k, -1, dtype=np.int64)
        for gid, g in enumerate(groups):
            if np.any(group_of[g] != -1):
                raise ValueError("groups must be pairwise disjoint")
            group_of[g] = gid
        if np.any(group_of < 0):
            raise ValueError("groups must cover every column index")
        if weights is None:
            weights = np.sqrt([g.size for g in groups])
        weights = np.array(weights, dtype=np.float64)
        if weights.shape != (len(groups),) or np.any(weights <= 0):
            raise ValueError("need one strictly positive weight per group")
        if spectral_norms is None:
            spectral_norms = group_spectral_norms(dictionary, groups)
        norms = np.asarray(spectral_norms, dtype=np.float64)
        sizes = np.array([g.size for g in groups], dtype=np.int64)
        offsets = np.concatenate(([0], np.cumsum(sizes)[:-1]))
        order = np.concatenate(groups)
        for arr in (weights, norms, group_of, order, offsets, *groups):
            arr.setflags(write=False)
        return cls(groups, weights, norms, group_of, order, offsets)

    @property
    def n_groups(self):
        return len(self.groups)

    @property
    def size(self):
        return self.group_of.size

    def group_sizes(self):
        return np.array([g.size for g in self.groups], dtype=np.int64)


@dataclass(frozen=True)
class Problem:
    """``min_x 1/2||Dx - y||^2 + lam * penalty(x)`` (problems.py:20-57)."""

    dictionary: Dictionary
    y: np.ndarray
    lam: float
    partition: GroupPartition | None = None

    def __post_init__(self):
        y = np.asarray(self.y, dtype=np.float64)
        if y.shape != (self.dictionary.n_rows,):
            raise ValueError("observation length must match the dictionary rows")
        nrm = float(np.linalg.norm(y))
        if abs(nrm - 1.0) > OBS_NORM_TOL:
            raise ValueError(f"observation must have unit l2 norm (got {nrm!r})")
        if not self.lam > 0:
            raise ValueError("lam must be strictly positive")
        if self.partition is not None and self.partition.size != self.dictionary.n_cols:
            raise ValueError("partition must cover exactly the dictionary columns")
        object.__setattr__(self, "y", y)
        object.__setattr__(self, "lam", float(self.lam))

    @property
    def kind(self):
        return LASSO if self.partition is None else GROUP

    @property
    def n_rows(self):
        return self.dictionary.n_rows

    @property
    def n_cols(self):
        return self.dictionary.n_cols


@dataclass(frozen=True)
class LambdaMax:
    """Trivial-solution threshold and its maximiser (problems.py:61-72)."""

    value: float
    atom: np.ndarray | None = None
    atom_index: int | None = None
    group: int | None = None


def expand(x_reduced, kept, k):
    """Scatter a reduced vector to the K original positions (problems.py:169-177)."""
    x_reduced = np.asarray(x_reduced, dtype=np.float64)
    kept = index_set(kept, k)
    if x_reduced.shape != (kept.size,):
        raise ValueError("reduced vector length must equal the kept index count")
    out = np.zeros(int(k), dtype=np.float64)
    out[kept] = x_reduced
    return out
