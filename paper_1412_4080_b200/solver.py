"""``run(problem, cfg, iteration_hook=None)`` on the B200 engine.

Mirrors the reference driver ``solvers.run`` (solvers.py:358-511): same config
fields and validation messages, same ``SolveResult`` / ``SolveTrace`` /
``ScreenState`` contents, same exception types.  The whole solve runs on the
device: one setup-graph launch plus one conditional-WHILE graph launch; the
host synchronises once at the end.  With an ``iteration_hook`` the engine is
stepped one iteration per launch and the pre-reduction snapshot
(``IterationInfo``, solvers.py:106-117) is copied back for the hook.

BASELINE extension: ``SolverConfig.gap_tol`` stops at the first iteration whose
duality gap ``F(x_t) - 1/2||y||^2 + lam^2/2 r_SAFE,t^2`` is <= gap_tol.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .instrument import (DYNAMIC, NONE, STATIC, STRATEGIES, SolveTrace, flops_iteration, flops_static_init,
                         problem_digest)
from .problem import GROUP, LASSO, LambdaMax, Problem

ISTA, FISTA, TWIST, SPARSA, CP = "ista", "fista", "twist", "sparsa", "cp"
ALGORITHMS = (ISTA, FISTA, TWIST, SPARSA, CP)
SAFE, DST3, DOME, GSAFE, GST3 = "safe", "dst3", "dome", "gsafe", "gst3"
LASSO_TESTS = (SAFE, DST3, DOME)
GROUP_TESTS = (GSAFE, GST3)


@dataclass
class SolverConfig:
    """Solver knobs (solvers.py:44-85) + ``gap_tol`` and an optional ``op_norm``."""

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
    op_norm: float | None = None

    def validate(self, kind):
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if self.strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {self.strategy!r}")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if not self.rel_tol > 0:
            raise ValueError("rel_tol must be positive")
        if not self.backtrack_factor > 1:
            raise ValueError("backtrack_factor must exceed 1")
        if not self.L0 > 0:
            raise ValueError("L0 must be positive")
        if not 0 < self.cp_step_safety < 1:
            raise ValueError("cp_step_safety must lie in (0, 1)")
        if self.strategy != NONE:
            allowed = LASSO_TESTS if kind == LASSO else GROUP_TESTS
            if self.test is None:
                raise ValueError("screening strategies require a test kind")
            if self.test not in allowed:
                raise ValueError(f"test {self.test!r} does not apply to {kind} problems")


@dataclass(frozen=True)
class ScreenState:
    """Monotone eliminated/kept index sets (screening.py:84-101)."""

    eliminated: np.ndarray
    kept: np.ndarray
    test_kind: str | None = None

    @classmethod
    def initial(cls, k, test_kind=None):
        return cls(np.empty(0, dtype=np.int64), np.arange(k, dtype=np.int64), test_kind)

    @property
    def size(self):
        return self.eliminated.size + self.kept.size


@dataclass
class IterationInfo:
    """Pre-reduction snapshot handed to an iteration hook (solvers.py:106-117)."""

    t: int
    theta: np.ndarray
    corr: np.ndarray
    kept: np.ndarray
    kept_groups: np.ndarray | None
    mask: np.ndarray | None
    x: np.ndarray
    context: object | None
    problem: object
    radius: float = float("nan")


@dataclass
class SolveResult:
    """Outcome of a run; ``x_star`` is expanded to the original indexing (solvers.py:121-132)."""

    x_star: np.ndarray
    iterations: int
    trace: SolveTrace
    final_objective: float
    screen_state: ScreenState
    lambda_max: float = float("nan")
    gap: float = float("nan")
    stop_reason: str = ""
    device_seconds: float = float("nan")

    @property
    def screened_fraction(self):
        return self.screen_state.eliminated.size / self.screen_state.size


@dataclass
class DeviceContext:
    """Host view of the per-solve precomputed correlations (ScreeningContext, screening.py:168-255)."""

    y_corr: np.ndarray
    star_corr: np.ndarray | None
    center_corr: np.ndarray | None
    center_group_norms: np.ndarray | None
    lmax: LambdaMax


_STOP_NAMES = {nat.STOP_RELTOL: "rel_tol", nat.STOP_GAP: "gap", nat.STOP_MAXITER: "max_iters",
               nat.STOP_EMPTY: "empty", nat.STOP_TRIVIAL: "trivial", nat.STOP_ERROR: "error"}


def _partition_key(part):
    """Content key of a GroupPartition (group order, sizes, weights, spectral norms): device
    arrays cached on the Dictionary are shared only by partitions with equal content, never by
    object identity (an id() can be recycled by a new partition)."""
    if part is None:
        return None
    import hashlib
    h = hashlib.sha1()
    for arr in (np.concatenate(part.groups).astype(np.int64), part.group_sizes(),
                np.asarray(part.weights, dtype=np.float64), np.asarray(part.spectral_norms, dtype=np.float64)):
        h.update(np.ascontiguousarray(arr).tobytes())
        h.update(b"|")
    return h.hexdigest()


class _DeviceDictionary:
    """Device arrays that depend only on the dictionary and the partition content (cached on
    the Dictionary, shared by every Problem / Engine on it): the padded column-major D
    (group-permuted), the group pointer, weights and spectral norms."""

    def __init__(self, dic, part, device):
        import torch
        self.n, self.k, self.ldd = dic.n_rows, dic.n_cols, dic.ldd
        self.perm = None
        self.group_ptr = self.group_w = self.group_sn = None
        self.n_groups = 0
        if part is not None:
            order = np.concatenate(part.groups)
            if not np.array_equal(order, np.arange(self.k)):
                self.perm = order.astype(np.int64)      # permuted column j -> original perm[j]
            sizes = part.group_sizes()
            ptr = np.concatenate(([0], np.cumsum(sizes))).astype(np.int32)
            self.group_ptr = torch.from_numpy(ptr).to(device)
            self.group_w = torch.from_numpy(np.array(part.weights, dtype=np.float64)).to(device)
            self.group_sn = torch.from_numpy(np.array(part.spectral_norms, dtype=np.float64)).to(device)
            self.n_groups = part.n_groups
            self.group_ptr_host = ptr
        self.D = dic.device_data(device, self.perm)
        self.col_norms = None
        if dic.norm_aware:
            # ||d_j|| of the stored (rounded) columns, a property of D alone: computed once per
            # dictionary upload instead of in every solve's setup (8.6 GB pass on c4)
            self.col_norms = torch.empty(self.k, dtype=torch.float64, device=device)
            L = nat.lib()
            nat.check(L.dscr_column_norms(dic.dtype_code, self.D.data_ptr(), self.ldd, self.n, self.k,
                                          self.col_norms.data_ptr(), nat.stream_ptr()))


class _DeviceProblem:
    """One Problem on the device: the cached dictionary arrays plus this problem's own
    observation, uploaded into a fresh buffer for every Engine (never cached: two Problems on
    one Dictionary carry different y)."""

    def __init__(self, problem, device):
        import torch
        dic = problem.dictionary
        cache = dic.__dict__.setdefault("_problem_cache", {})
        key = (str(device), _partition_key(problem.partition))
        dd = cache.get(key)
        if dd is None:
            dd = _DeviceDictionary(dic, problem.partition, device)
            cache[key] = dd
        self.dd = dd
        self.n, self.k, self.ldd = dd.n, dd.k, dd.ldd
        self.perm, self.n_groups, self.D = dd.perm, dd.n_groups, dd.D
        self.group_ptr, self.group_w, self.group_sn = dd.group_ptr, dd.group_w, dd.group_sn
        self.col_norms = dd.col_norms
        if dd.n_groups:
            self.group_ptr_host = dd.group_ptr_host
        y = torch.zeros(self.ldd, dtype=torch.float64)
        y[: self.n] = torch.from_numpy(problem.y)
        self.y = y.to(device, non_blocking=True)


def _desc(problem, dp):
    d = nat.ProblemDesc()
    d.dtype = problem.dictionary.dtype_code
    d.n_rows, d.n_cols, d.ldd = dp.n, dp.k, dp.ldd
    d.D, d.y = dp.D.data_ptr(), dp.y.data_ptr()
    d.lam = problem.lam
    d.n_groups = dp.n_groups
    dic = problem.dictionary
    d.norm_aware = int(dic.norm_aware)
    if dp.n_groups:
        d.group_ptr, d.group_w, d.group_snorm = dp.group_ptr.data_ptr(), dp.group_w.data_ptr(), dp.group_sn.data_ptr()
    d.col_offset, d.n_cols_total = 0, dp.k
    d.group_offset, d.n_groups_total = 0, dp.n_groups
    d.col_norms = dp.col_norms.data_ptr() if dp.col_norms is not None else None
    return d


def _config(cfg, op_norm):
    c = nat.Config()
    c.algorithm = nat.ALGO_CODES[cfg.algorithm]
    c.strategy = nat.STRATEGY_CODES[cfg.strategy]
    c.test = nat.TEST_CODES[cfg.test] if cfg.strategy != NONE else -1
    c.max_iters = int(cfg.max_iters)
    c.rel_tol = float(cfg.rel_tol)
    c.gap_tol = float(cfg.gap_tol) if cfg.gap_tol is not None else -1.0
    c.L0 = float(cfg.L0)
    c.backtrack_factor = float(cfg.backtrack_factor)
    c.twist_alpha, c.twist_beta = float(cfg.twist_alpha), float(cfg.twist_beta)
    c.twist_step = float(cfg.twist_step) if cfg.twist_step is not None else -1.0
    c.cp_gamma, c.cp_step_safety = float(cfg.cp_gamma), float(cfg.cp_step_safety)
    c.bb_L_min, c.bb_L_max = float(cfg.bb_L_min), float(cfg.bb_L_max)
    c.op_norm = float(op_norm) if op_norm is not None else -1.0
    return c


class Engine:
    """One solver handle on the device: workspace, graphs, readback helpers."""

    def __init__(self, problem, cfg, device=None, stream=None, desc_patch=None):
        import torch
        self.torch = torch
        self.problem, self.cfg = problem, cfg
        self.L = nat.lib()
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.sptr = C.c_void_p(self.stream.cuda_stream)
        dic = problem.dictionary
        with torch.cuda.stream(self.stream):
            dp = _DeviceProblem(problem, self.device)
            self.dp = dp
            op_norm = cfg.op_norm
            need_norm = cfg.algorithm == CP or (cfg.algorithm == TWIST and cfg.twist_step is None)
            if need_norm and op_norm is None:
                if dic._op_norm is None:
                    from .problem import operator_norm
                    dic._op_norm = operator_norm(dic)
                op_norm = dic._op_norm
                if op_norm <= 0:
                    raise ValueError("dictionary has zero operator norm")
            if cfg.algorithm == CP and op_norm is not None:
                tau = cfg.cp_step_safety / op_norm
                if tau * tau * op_norm ** 2 >= 1.0:
                    raise ValueError("primal-dual step sizes violate tau*sigma*||D||^2 < 1")
            self.desc = _desc(problem, dp)
            for key, val in (desc_patch or {}).items():
                setattr(self.desc, key, val)
            self.ccfg = _config(cfg, op_norm)
            nbytes = int(self.L.dscr_solver_workspace_size(C.byref(self.desc), C.byref(self.ccfg)))
            if nbytes == 0:
                nat.check(nat.DSCR_EINVAL if not self.L.dscr_last_error() else -1, "workspace size")
            self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            h = C.c_void_p()
            nat.check(self.L.dscr_solver_create(C.byref(self.desc), C.byref(self.ccfg), self.ws.data_ptr(),
                                                nbytes, self.sptr, C.byref(h)))
            self.h = h
            self.bufs = nat.Buffers()
            nat.check(self.L.dscr_solver_get_buffers(self.h, C.byref(self.bufs)))

    def close(self):
        if getattr(self, "h", None):
            self.stream.synchronize()
            self.L.dscr_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- driving -----------------------------------------------------------
    def setup(self):
        nat.check(self.L.dscr_solver_setup(self.h, self.sptr))

    def launch(self, limit=0):
        nat.check(self.L.dscr_solver_run(self.h, int(limit), self.sptr))

    def scalars(self):
        s = nat.Scalars()
        nat.check(self.L.dscr_solver_scalars(self.h, self.sptr, C.byref(s)))
        return s

    # -- typed views into the workspace ------------------------------------
    def view(self, ptr, count, dtype):
        torch = self.torch
        isz = torch.empty((), dtype=dtype).element_size()
        off = int(ptr) - self.ws.data_ptr()
        return self.ws[off: off + count * isz].view(dtype)

    def active_units(self, parity):
        """Flat active unit list (ordered) of the given parity buffer, on the host."""
        torch = self.torch
        b = self.bufs
        G, cap = b.G, b.cap
        cnt = self.view(b.act_cnt[parity], G, torch.int32).cpu().numpy()
        lst = self.view(b.act[parity], G * cap, torch.int32).cpu().numpy().reshape(G, cap)
        return np.concatenate([lst[s, : cnt[s]] for s in range(G)]) if G else np.empty(0, np.int32)

    def vec(self, ptr, count):
        return self.view(ptr, count, self.torch.float64).cpu().numpy()

    def trace_rows(self, t):
        if t <= 0:
            return np.zeros((0, nat.TRACE_FIELDS))
        return self.vec(self.bufs.trace, t * nat.TRACE_FIELDS).reshape(t, nat.TRACE_FIELDS)

    def units_to_atoms(self, units):
        """Local (permuted) column indices of the given units."""
        if self.dp.n_groups == 0:
            return np.asarray(units, dtype=np.int64)
        ptr = self.dp.group_ptr_host
        return np.concatenate([np.arange(ptr[u], ptr[u + 1]) for u in units]).astype(np.int64) \
            if len(units) else np.empty(0, np.int64)

    def to_original(self, cols):
        cols = np.asarray(cols, dtype=np.int64)
        return cols if self.dp.perm is None else self.dp.perm[cols]


def _raise_status(L, sc):
    if sc.status == nat.DSCR_ENONFINITE:
        raise FloatingPointError("solver produced a non-finite iterate (or backtracking failed to find a valid step)")
    if sc.status == nat.DSCR_ERADIUS:
        raise RuntimeError("squared screening radius fell below the guard; region construction is inconsistent")
    if sc.status != 0:
        raise RuntimeError(f"solver failed with status {sc.status}")


def _context(eng, sc):
    b = eng.bufs
    k = eng.dp.k
    inv = np.empty(k, dtype=np.int64)
    perm = eng.dp.perm
    if perm is not None:
        inv[perm] = np.arange(k)

    def orig(v):
        return v if perm is None else v[inv]

    ycorr = orig(eng.vec(b.y_corr, k))
    test = eng.cfg.test
    star = orig(eng.vec(b.star_corr, k)) if test in (DST3, DOME) else None
    cc = orig(eng.vec(b.cc, k)) if eng.cfg.strategy != NONE else None
    cn = eng.vec(b.cnorm, eng.dp.n_groups) if eng.dp.n_groups and eng.cfg.strategy != NONE else None
    if eng.dp.n_groups:
        lm = LambdaMax(float(sc.lmax), group=int(sc.lmax_index))
    else:
        lm = LambdaMax(float(sc.lmax), atom=sc.lmax_sign * eng.problem.dictionary.column(int(sc.lmax_index)),
                       atom_index=int(sc.lmax_index))
    return DeviceContext(ycorr, star, cc, cn, lm)


def _hook_info(eng, sc_after, t):
    """IterationInfo of the iteration that just completed (pre-reduction view)."""
    b = eng.bufs
    p_old = sc_after.parity ^ 1
    units_old = eng.active_units(p_old)
    atoms_old = eng.units_to_atoms(units_old)
    orig = eng.to_original(atoms_old)
    order = np.argsort(orig, kind="stable")
    kept = orig[order]
    k = eng.dp.k
    theta = eng.vec(b.theta[p_old], eng.dp.n)
    corr = eng.vec(b.corr, k)[atoms_old][order]
    x = eng.vec(b.x[sc_after.xi], k)[atoms_old][order]
    mask = None
    if eng.cfg.strategy == DYNAMIC:
        um = eng.view(b.mask, len(units_old), eng.torch.uint8).cpu().numpy().astype(bool)
        if eng.dp.n_groups:
            sizes = np.diff(eng.dp.group_ptr_host)[units_old]
            mask = np.repeat(um, sizes)[order]
        else:
            mask = um[order]
    kept_groups = np.sort(units_old.astype(np.int64)) if eng.dp.n_groups else None
    return IterationInfo(t=t, theta=theta, corr=corr, kept=kept, kept_groups=kept_groups, mask=mask, x=x,
                         context=None, problem=eng.problem, radius=float(sc_after.radius))


def run(problem, cfg, iteration_hook=None, device=None, stream=None):
    """Solve ``problem`` with the configured algorithm and screening strategy on the GPU."""
    if not isinstance(problem, Problem):
        raise TypeError("problem must be a paper_1412_4080_b200.Problem")
    cfg.validate(problem.kind)
    eng = Engine(problem, cfg, device=device, stream=stream)
    try:
        return _solve(eng, problem, cfg, iteration_hook)
    finally:
        eng.close()


def _solve(eng, problem, cfg, iteration_hook):
    k, n = problem.n_cols, problem.n_rows
    group_count = problem.partition.n_groups if problem.kind == GROUP else 0
    start = eng.torch.cuda.Event(enable_timing=True)
    stop = eng.torch.cuda.Event(enable_timing=True)
    start.record(eng.stream)
    eng.setup()
    if iteration_hook is None:
        eng.launch(0)
        stop.record(eng.stream)
        sc = eng.scalars()
    else:
        sc = eng.scalars()
        ctx = _context(eng, sc) if sc.stop != nat.STOP_TRIVIAL and sc.stop != nat.STOP_ERROR else None
        while sc.stop == nat.STOP_RUNNING:
            t_before = sc.t
            eng.launch(t_before + 1)
            sc = eng.scalars()
            if sc.t == t_before:
                break
            info = _hook_info(eng, sc, sc.t)
            info.context = ctx
            iteration_hook(info)
        stop.record(eng.stream)
        eng.stream.synchronize()
    _raise_status(eng.L, sc)
    device_s = start.elapsed_time(stop) / 1e3 if iteration_hook is None else float("nan")
    trace = SolveTrace(kind=problem.kind, strategy=cfg.strategy, n_rows=n, n_cols=k,
                       group_count=group_count, lam=problem.lam, digest=problem_digest(problem))
    if sc.trivial:
        st = ScreenState(np.arange(k, dtype=np.int64), np.empty(0, dtype=np.int64), cfg.test)
        return SolveResult(np.zeros(k), 0, trace, 0.5 * float(problem.y @ problem.y), st,
                           lambda_max=float(sc.lmax), stop_reason="trivial", device_seconds=device_s)
    t = int(sc.t)
    rows = eng.trace_rows(t)
    cum = 0
    if cfg.strategy == STATIC:
        trace.init_flops = flops_static_init(k, n)
        cum = trace.init_flops
    for r in rows:
        cum += flops_iteration(problem.kind, cfg.strategy, k, n, int(r[nat.TR_KEPT]), int(r[nat.TR_NNZ]),
                               group_count)
        trace.append(int(r[nat.TR_T]), int(r[nat.TR_KEPT]), int(r[nat.TR_NNZ]), float(r[nat.TR_OBJ]), cum,
                     float(r[nat.TR_NS]) * 1e-9)
        trace.gap.append(float(r[nat.TR_GAP]))
        trace.radius.append(float(r[nat.TR_RADIUS]))
        trace.support.append(int(r[nat.TR_SUPPORT]))
        trace.L.append(float(r[nat.TR_L]))
    units = eng.active_units(sc.parity)
    atoms = eng.units_to_atoms(units)
    xs = eng.vec(eng.bufs.x[sc.xi], k)[atoms]
    kept = eng.to_original(atoms)
    order = np.argsort(kept, kind="stable")
    kept = kept[order]
    x_star = np.zeros(k)
    x_star[kept] = xs[order]
    mask = np.ones(k, dtype=bool)
    mask[kept] = False
    elim = np.flatnonzero(mask).astype(np.int64)
    final = trace.objective[-1] if trace.objective else 0.5 * float(problem.y @ problem.y)
    return SolveResult(x_star, t, trace, final, ScreenState(elim, kept.astype(np.int64), cfg.test),
                       lambda_max=float(sc.lmax), gap=float(sc.gap) if t else float("nan"),
                       stop_reason=_STOP_NAMES.get(sc.stop, "running"), device_seconds=device_s)
