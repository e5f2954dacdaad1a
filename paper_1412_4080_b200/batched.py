"""Batched many-observation Lasso (BASELINE config 5, the dictionary-learning inner step).

``solve_batched`` runs FISTA with per-observation dynamic screening for a batch
of observations sharing one bf16 dictionary.  Each observation is the
reference's single-observation problem (``solvers.run`` with FISTA, a fixed
step 1/L and the SAFE or DST3 test); the batch turns the per-observation
correlations ``D^T theta_j`` into one tensor-core contraction (tcgen05, bf16
in / fp32 accumulate) and keeps the iterates sparse per observation.

Differences from the reference's per-observation run, all documented in
DESIGN.md: the step is fixed (no backtracking test; BASELINE: step 1/||D||^2),
the correlations carry bf16/fp32 error, and the dual-scaling bound is inflated
by a rigorous bound on that error so the screening stays safe.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat


class BatchedCapacityError(RuntimeError):
    """An observation had more hot correlations than the fused epilogue's per-observation list
    (2048) or more nonzeros than ``cap``; solve_batched / BatchedSolver retry once on the dense
    path with ``cap`` = the atom count."""


_PAD_LAM = 1e30      # lam of the padding observations: above any lambda_*, so they are trivial (status 1)


def fista_betas(iters):
    """Momentum coefficients (l_t - 1)/l_{t+1} of solvers.py:216-218, same fp64 ops."""
    out = np.empty(iters)
    l_acc = 1.0
    for t in range(iters):
        l_new = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * l_acc ** 2))
        out[t] = (l_acc - 1.0) / l_new
        l_acc = float(l_new)
    return out


@dataclass
class BatchedResult:
    iterations: int
    objective: np.ndarray        # F_j per observation after the last iteration
    gap: np.ndarray
    nnz: np.ndarray
    kept: np.ndarray
    status: np.ndarray           # 0 ok, 1 trivial (lam_j > lambda_*), 3 radius guard, 4 capacity
    lambda_max: np.ndarray
    radius: np.ndarray
    trace: np.ndarray            # [iterations][4]: sum F, sum gap, sum nnz, sum kept
    x_ptr: np.ndarray            # CSR over observations: x_j = (x_indices, x_values)[x_ptr[j]:x_ptr[j+1]]
    x_indices: np.ndarray
    x_values: np.ndarray
    device_seconds: float = float("nan")
    d2h_bytes: int = 0           # bytes copied device -> host by result()
    active_words: np.ndarray | None = None   # [B][K/32] active-atom bits (result(masks=True) only)
    n_atoms: int | None = None               # the caller's atom count (the device pads it to a multiple of 128)

    def active_mask(self, j):
        """Boolean active-atom mask of observation j (needs the masks read back)."""
        if self.active_words is None:
            raise ValueError("masks were not read back (solve_batched(..., masks=True))")
        bits = np.unpackbits(self.active_words[j].view(np.uint8), bitorder="little")
        return bits.astype(bool)[:self.n_atoms]

    def eliminated(self, j):
        """Atoms screened out of observation j (sorted)."""
        return np.flatnonzero(~self.active_mask(j)).astype(np.int64)

    @property
    def x_idx(self):
        """Per-observation support (sorted atom indices), split from the CSR arrays on first use."""
        if not hasattr(self, "_x_idx"):
            self._x_idx = np.split(self.x_indices, self.x_ptr[1:-1])
        return self._x_idx

    @property
    def x_val(self):
        if not hasattr(self, "_x_val"):
            self._x_val = np.split(self.x_values, self.x_ptr[1:-1])
        return self._x_val

    def x_dense(self, j, k):
        out = np.zeros(k)
        out[self.x_idx[j]] = self.x_val[j]
        return out


class BatchedEngine:
    """Device state of one batch: workspace, handle, graph."""

    def __init__(self, dictionary, Y, lam, L, iterations=100, test="dst3", splits=1, cap=1024, device=None,
                 fused=True):
        import torch
        if dictionary.dtype != "bf16":
            raise ValueError("the batched path takes a bf16 dictionary (Dictionary(..., dtype='bf16'))")
        y_torch = torch.is_tensor(Y)          # e.g. the transposed view of a pinned (b, n) host buffer
        if y_torch:
            if Y.dtype != torch.float64 or Y.dim() != 2 or Y.device.type != "cpu":
                raise ValueError("observations must be a 2-D float64 host tensor or array")
        else:
            Y = np.asarray(Y, dtype=np.float64)
        n, b = Y.shape
        if n != dictionary.n_rows:
            raise ValueError("observations must have the dictionary's row count")
        lam = np.asarray(lam, dtype=np.float64).reshape(-1)
        if lam.shape != (b,) or np.any(lam <= 0):
            raise ValueError("need one strictly positive lam per observation")
        self.torch = torch
        self.L = nat.lib()
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        # The kernels take N % 64 == 0, K % 128 == 0, B % 256 == 0 (tile shapes).  Other shapes are
        # padded here: zero rows (no contribution to any product), all-zero atoms (never active:
        # the kernels drop them from the masks and the kept counts) and trivial observations
        # (a copy of observation 0 with lam > lambda_*: status 1, skipped by every kernel and by
        # the batch aggregates); results are cut back to the caller's shapes.
        self.k_user, self.n_user, self.b_user = dictionary.n_cols, n, b
        kp, np_, bp = (dictionary.n_cols + 127) // 128 * 128, (n + 63) // 64 * 64, (b + 255) // 256 * 256
        self.k, self.n, self.b = kp, np_, bp
        self.iterations, self.cap = int(iterations), int(cap)
        self.Dt_src = dictionary.device_data(self.device)                  # (K, ldd) bf16 bits
        self.dic = dictionary
        if kp != dictionary.n_cols or np_ > dictionary.ldd:
            self.Dt = torch.zeros((kp, np_), dtype=self.Dt_src.dtype, device=self.device)
            self.Dt[:dictionary.n_cols, :min(dictionary.ldd, np_)].copy_(self.Dt_src[:, :min(dictionary.ldd, np_)])
            ldd = np_
        else:
            self.Dt, ldd = self.Dt_src, dictionary.ldd
        ldy = np_
        # upload Y as given (n x b) and transpose on the device into observation rows [b][ldy]
        self.Yd = torch.zeros((bp, ldy), dtype=torch.float64, device=self.device)
        if y_torch:
            rows = Y.T if Y.T.is_contiguous() else Y.T.contiguous()              # (b, n)
            self.Yd[:b, :n].copy_(rows.to(self.device, non_blocking=rows.is_pinned()))
            y_bytes = int(Y.numel() * 8)
        else:
            Yh = torch.from_numpy(Y.T if Y.flags.f_contiguous else np.ascontiguousarray(Y))
            if Y.flags.f_contiguous:
                self.Yd[:b, :n].copy_(Yh.to(self.device))
            else:
                self.Yd[:b, :n].copy_(Yh.to(self.device).T)
            y_bytes = int(Y.nbytes)
        self.lamd = torch.full((bp,), _PAD_LAM, dtype=torch.float64, device=self.device)
        self.lamd[:b].copy_(torch.from_numpy(lam.copy()))
        if bp != b:
            self.Yd[b:].copy_(self.Yd[0:1].expand(bp - b, ldy))
        self.h2d_bytes = int(y_bytes + lam.nbytes)
        self.betas = fista_betas(self.iterations)
        d = nat.BatchedDesc()
        d.n_rows, d.n_atoms, d.n_obs, d.ldd = np_, kp, bp, ldd
        d.Dt, d.Y, d.ldy, d.splits = self.Dt.data_ptr(), self.Yd.data_ptr(), ldy, int(splits)
        d.lam, d.L, d.test, d.cap = self.lamd.data_ptr(), float(L), nat.TEST_CODES[test], self.cap
        d.max_iters = self.iterations
        d.fused = 1 if fused else 0
        d.beta = self.betas.ctypes.data
        self.desc = d
        nbytes = int(self.L.dscr_batched_workspace_size(C.byref(d)))
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.stream = torch.cuda.current_stream(self.device)
        self.sptr = C.c_void_p(self.stream.cuda_stream)
        h = C.c_void_p()
        nat.check(self.L.dscr_batched_create(C.byref(d), self.ws.data_ptr(), nbytes, self.sptr, C.byref(h)))
        self.h = h
        self.bufs = nat.BatchedBuffers()
        nat.check(self.L.dscr_batched_get_buffers(self.h, C.byref(self.bufs)))

    def dic_current(self):
        """The dictionary's device copy is still the one in this engine's buffer (it is not when
        the caller dropped the device copy, e.g. after updating the host data)."""
        return any(t.data_ptr() == self.Dt_src.data_ptr() for t in self.dic._dev.values())

    def load(self, Y, lam):
        """New observations and lambdas of the same shape for another solve on this engine (the
        workspace, the captured iteration graph and the device dictionary are reused)."""
        torch = self.torch
        lam = np.asarray(lam, dtype=np.float64).reshape(-1)
        b = self.b_user
        if lam.shape != (b,) or np.any(lam <= 0):
            raise ValueError("need one strictly positive lam per observation")
        n = self.n_user
        if torch.is_tensor(Y):
            if Y.dtype != torch.float64 or tuple(Y.shape) != (n, b) or Y.device.type != "cpu":
                raise ValueError("observations must be a float64 host tensor of shape (n_rows, batch)")
            rows = Y.T if Y.T.is_contiguous() else Y.T.contiguous()
            self.Yd[:b, :n].copy_(rows.to(self.device, non_blocking=rows.is_pinned()))
            y_bytes = int(Y.numel() * 8)
        else:
            Y = np.asarray(Y, dtype=np.float64)
            if Y.shape != (n, b):
                raise ValueError("observations must have shape (n_rows, batch)")
            Yh = torch.from_numpy(Y.T if Y.flags.f_contiguous else np.ascontiguousarray(Y))
            if Y.flags.f_contiguous:
                self.Yd[:b, :n].copy_(Yh.to(self.device))
            else:
                self.Yd[:b, :n].copy_(Yh.to(self.device).T)
            y_bytes = int(Y.nbytes)
        if self.b != b:
            self.Yd[b:].copy_(self.Yd[0:1].expand(self.b - b, self.Yd.shape[1]))
        self.lamd[:b].copy_(torch.from_numpy(lam))
        self.h2d_bytes = int(y_bytes + lam.nbytes)

    def setup(self):
        nat.check(self.L.dscr_batched_setup(self.h, self.sptr))

    def run(self):
        nat.check(self.L.dscr_batched_run(self.h, self.iterations, self.sptr))

    def _view(self, ptr, count, dtype):
        torch = self.torch
        isz = torch.empty((), dtype=dtype).element_size()
        off = int(ptr) - self.ws.data_ptr()
        return self.ws[off: off + count * isz].view(dtype)

    def result(self, device_seconds=float("nan"), masks=False):
        """Copy the solution back: device-side CSR compaction of the x lists, then a few
        packed transfers (self.d2h_bytes counts them).  ``masks=True`` also reads the active-atom
        bit masks (B x K/32 words) for set-level checks."""
        torch = self.torch
        bp, b, bf, cap = self.b, self.b_user, self.bufs, self.cap      # padded / caller's batch size
        par = self.iterations & 1
        cnt = self._view(bf.s_cnt[par], bp, torch.int32)[:b]
        xs = self._view(bf.s_x[par], bp * cap, torch.float64).view(bp, cap)[:b]
        live = (torch.arange(cap, device=self.device, dtype=torch.int32)[None, :] < cnt[:, None]) & (xs != 0.0)
        counts_d = live.sum(dim=1, dtype=torch.int32)
        idx = self._view(bf.s_idx[par], bp * cap, torch.int32).view(bp, cap)[:b][live].cpu().numpy()
        val = xs[live].cpu().numpy()
        f64 = torch.stack([self._view(p, bp, torch.float64)[:b] for p in (bf.F, bf.gap, bf.lmax, bf.radius)]).cpu().numpy()
        i32 = torch.cat([self._view(p, bp, torch.int32)[:b] for p in (bf.nnz, bf.kept, bf.status)] + [counts_d]
                        + [self._view(bf.iterations, 1, torch.int32)]).cpu().numpy()
        trace = self._view(bf.trace, self.iterations * 4, torch.float64).cpu().numpy().reshape(-1, 4)
        words = None
        if masks:
            words = self._view(bf.mask, bp * (self.k // 32), torch.int32).view(bp, self.k // 32)[:b].cpu().numpy()
            words = words.view(np.uint32)
        self.d2h_bytes = int(idx.nbytes + val.nbytes + f64.nbytes + i32.nbytes + trace.nbytes
                             + (words.nbytes if words is not None else 0))
        nnz, kept, status, counts = (i32[q * b:(q + 1) * b] for q in range(4))
        if np.any(status >= 3):
            bad = np.flatnonzero(status >= 3)
            code = int(status[bad[0]])
            exc = BatchedCapacityError if np.all(status[bad] == 4) else RuntimeError
            raise exc(f"batched solve failed on {bad.size} observations (status {code}: "
                      f"{'radius guard' if code == 3 else 'nonzero capacity exceeded'})")
        ptr = np.zeros(b + 1, dtype=np.int64)
        np.cumsum(counts, out=ptr[1:])
        return BatchedResult(
            iterations=int(i32[4 * b]),
            objective=f64[0], gap=f64[1], nnz=nnz, kept=kept, status=status,
            lambda_max=f64[2], radius=f64[3], trace=trace,
            x_ptr=ptr, x_indices=idx.astype(np.int64), x_values=val,
            device_seconds=device_seconds, d2h_bytes=self.d2h_bytes, active_words=words, n_atoms=self.k_user,
        )

    def close(self):
        if getattr(self, "h", None):
            self.stream.synchronize()
            self.L.dscr_batched_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_batched(dictionary, Y, lam, L, iterations=100, test="dst3", splits=1, cap=1024, device=None,
                  fused=True, masks=False):
    """FISTA (fixed step 1/L) with per-observation dynamic screening for Y[:, j], lam[j].
    ``masks=True`` also returns the per-observation active-atom masks (``BatchedResult.eliminated``)."""
    def once(cap_, fused_):
        eng = BatchedEngine(dictionary, Y, lam, L, iterations, test, splits, cap_, device, fused_)
        torch = eng.torch
        try:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(eng.stream)
            eng.setup()
            eng.run()
            ev1.record(eng.stream)
            eng.stream.synchronize()
            return eng.result(ev0.elapsed_time(ev1) / 1e3, masks=masks)
        finally:
            eng.close()

    try:
        return once(cap, fused)
    except BatchedCapacityError:
        # the reference has no support-size limit: rerun with room for every atom, dense update
        return once((dictionary.n_cols + 127) // 128 * 128, False)


class BatchedSolver:
    """Repeated batched solves on one dictionary (the dictionary-learning inner loop): the
    engine -- workspace, captured iteration graph, device dictionary -- is built on the first
    solve and reused while the batch shape stays the same.

        solver = BatchedSolver(dictionary, L, iterations=100, test="dst3")
        for Y, lam in batches:
            res = solver.solve(Y, lam)
        solver.close()
    """

    def __init__(self, dictionary, L, iterations=100, test="dst3", splits=1, cap=1024, device=None, fused=True):
        self.args = (dictionary, L, iterations, test, splits, cap, device, fused)
        self.eng = None

    def solve(self, Y, lam, dictionary=None):
        """Solve one batch; `dictionary` (same shape and dtype) replaces the dictionary first,
        e.g. after a dictionary-learning update (uploaded into the engine's buffer)."""
        d0, L, iterations, test, splits, cap, device, fused = self.args
        if dictionary is not None:
            if (dictionary.n_rows, dictionary.n_cols, dictionary.dtype) != (d0.n_rows, d0.n_cols, d0.dtype):
                raise ValueError("a replacement dictionary must keep the shape and dtype")
            self.args = (dictionary,) + self.args[1:]
        dictionary = self.args[0]
        shape = tuple(Y.shape)
        if self.eng is not None and (self.eng.n_user, self.eng.b_user) == shape:
            if (self.eng.dic is not dictionary or not self.eng.dic_current()) and self.eng.Dt is not self.eng.Dt_src:
                # padded engine buffer: the dictionary keeps its own device copy, the engine's
                # padded buffer is refreshed from it
                fresh = dictionary.device_data(self.eng.device)          # upload (H2D) if not cached
                ld = min(dictionary.ldd, self.eng.Dt.shape[1])
                self.eng.Dt[:dictionary.n_cols, :ld].copy_(fresh[:, :ld])
                self.eng.Dt_src = fresh
                self.eng.dic = dictionary
            elif self.eng.dic is not dictionary or not self.eng.dic_current():
                prev = self.eng.dic                                      # its cache must not alias the buffer
                for key in [k for k, t in prev._dev.items() if t.data_ptr() == self.eng.Dt.data_ptr()]:
                    del prev._dev[key]
                fresh = dictionary.device_data(self.eng.device)          # upload (H2D)
                self.eng.Dt.copy_(fresh)
                dictionary.drop_device()
                dictionary._dev[(str(self.eng.device), None)] = self.eng.Dt   # the engine's buffer is the copy
                self.eng.Dt_src = self.eng.Dt
                self.eng.dic = dictionary
            self.eng.load(Y, lam)
        else:
            self.close()
            self.eng = BatchedEngine(dictionary, Y, lam, L, iterations, test, splits, cap, device, fused)
        eng = self.eng
        torch = eng.torch
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(eng.stream)
        eng.setup()
        eng.run()
        ev1.record(eng.stream)
        eng.stream.synchronize()
        try:
            return eng.result(ev0.elapsed_time(ev1) / 1e3)
        except BatchedCapacityError:
            # rebuild the engine with room for every atom and the dense update, and keep it
            self.close()
            self.args = (dictionary, L, iterations, test, splits, (dictionary.n_cols + 127) // 128 * 128, device, False)
            return self.solve(Y, lam)

    def close(self):
        if self.eng is not None:
            self.eng.close()
            self.eng = None
