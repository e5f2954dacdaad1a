"""TEST-ONLY numpy phase backend for paper_1412_4080_b200.dist.orchestrate.

Mirrors, phase by phase, what the CUDA engine does on one rank's column block
(K1 correlations/update, K1R radius from the MAX-reduced bound, K2 test and
reduction, K3A/K3S partial residuals, K3B finalize + epilogue; with one collective per trip K2S support
before the test, rank-slot gather, K1R1 radius / dropped / all-screened flags,
K2C test and compaction), so the
multi-rank orchestration (collective sequence, lambda_* argmax, owner
broadcast, stop/redo/fixup control) can run under gloo on CPU and be compared
with the unsharded oracle.  Lasso problems; ISTA, FISTA, SpaRSA, CP; SAFE/DST3.
"""

from __future__ import annotations

import numpy as np
import torch

from paper_1412_4080_b200 import _native as nat

STOP_RUNNING = 0


class _Scalars:
    pass


class NumpyShard:
    def __init__(self, D_local, y, lam, cfg, col_offset, op_norm=None):
        self.D = np.asfortranarray(D_local)
        self.y = np.asarray(y, dtype=np.float64)
        self.lam = float(lam)
        self.cfg = cfg
        self.unit_offset = col_offset
        self.n, self.k = self.D.shape
        self.ldd = self.n
        self.comm = torch.zeros(nat.CM_VEC + 2 * self.n + nat.OC_SLOT * nat.OC_MAX_WORLD, dtype=torch.float64)
        self.one = False
        self.rank, self.world = 0, 1
        self.vec = torch.zeros(self.n, dtype=torch.float64)
        self.op_norm = op_norm
        self.sc = _Scalars()

    # ---------------------------------------------------------------- helpers
    def _c(self):
        return self.comm.numpy()

    def scalars(self):
        return self.sc

    def set_collectives(self, rank, world, one):
        self.rank, self.world, self.one = rank, world, bool(one)

    def setup_peers(self, pg, rank, world):   # the device exchange is mirrored by a host SUM
        self.peer_pg = pg

    def _ph19(self):  # K3X_PUSH: nothing to stage on the host
        pass

    def _ph20(self):  # K3X_REDUCE: the SUM the device exchange computes (rank order)
        if self.sc.stop:
            return
        import torch.distributed as dist
        sec = self.comm[nat.CM_SUM: nat.CM_VEC + 2 * self.n + nat.OC_SLOT * self.world]
        if self.peer_pg is not None:
            parts = [torch.empty_like(sec) for _ in range(self.world)]
            dist.all_gather(parts, sec.clone(), group=self.peer_pg)
            acc = torch.zeros_like(sec)
            for part in parts:
                acc += part
            sec.copy_(acc)

    # ---------------------------------------------------------------- phases
    def phase(self, ph):
        getattr(self, "_ph%d" % ph)()

    def _ph0(self):  # SETUP_LOCAL
        sc, cfg = self.sc, self.cfg
        sc.t, sc.stop, sc.status, sc.mode, sc.trivial = 0, STOP_RUNNING, 0, 0, 0
        sc.L, sc.l_acc, sc.moved, sc.have_fprev, sc.f_prev = cfg.L0, 1.0, False, False, 0.0
        self.x = np.zeros(self.k)
        self.xp = np.zeros(self.k)
        self.u = np.zeros(self.k)
        self.active = np.arange(self.k)
        self.first = True
        if cfg.algorithm == "cp":
            sig = cfg.cp_step_safety / self.op_norm
            sc.tau = sc.sigma = sig
            self.theta = (0.0 + sig * (0.0 - self.y)) / (1.0 + sig)
        else:
            self.theta = 0.0 - self.y
        self.tw = (1.0 / self.op_norm ** 2) if cfg.algorithm == "twist" else None
        sc.yy = float(self.y @ self.y)
        sc.theta_sq = float(self.theta @ self.theta)
        sc.theta_y = float(self.theta @ self.y)
        self.ycorr = self.D.T @ self.y
        i = int(np.argmax(np.abs(self.ycorr)))
        c = self._c()
        c[nat.CM_SETUP:nat.CM_SETUP + 3] = [abs(self.ycorr[i]), i + self.unit_offset,
                                            1.0 if self.ycorr[i] >= 0 else -1.0]

    def _ph1(self):  # SETUP_ADOPT
        c = self._c()[nat.CM_SETUP:]
        sc = self.sc
        sc.lmax, sc.lmax_index, sc.lmax_sign = c[0], int(c[1]), c[2]
        self.owner_unit = int(c[6]) if c[4] > 0 else -1
        if c[3] > 0:
            sc.trivial, sc.stop = 1, 5

    def _ph2(self):  # SETUP_VEC (owner)
        self.vec[:] = torch.from_numpy(self.sc.lmax_sign * self.D[:, self.owner_unit])

    def _ph3(self):  # SETUP_FINISH
        if self.sc.stop:
            return
        sc, test = self.sc, self.cfg.test
        self.shift = sc.lmax / self.lam - 1.0
        safe = self.ycorr / self.lam
        if test == "dst3":
            star = self.D.T @ self.vec.numpy()
            self.cc = safe - self.shift * star
            sc.shift_sq = self.shift ** 2
        else:
            self.cc = safe
            sc.shift_sq = 0.0

    def _ph10(self):  # K1
        sc, cfg = self.sc, self.cfg
        if sc.stop or sc.mode == 2:
            return
        A = self.active
        if sc.mode == 0:
            self.corr = np.zeros(self.k)
            self.corr[A] = self.D[:, A].T @ self.theta
        c = self.corr[A]
        algo = cfg.algorithm
        if algo == "fista":
            point = self.u[A]
            v = point - c / sc.L
            thr = self.lam / sc.L
        elif algo == "cp":
            point = self.x[A]
            v = point - sc.tau * c
            thr = self.lam * sc.tau
        else:
            point = self.x[A]
            v = point - c / sc.L
            thr = self.lam / sc.L
        cand = np.sign(v) * np.maximum(np.abs(v) - thr, 0.0)
        self.xn = np.zeros(self.k)
        self.xn[A] = cand
        st = cand - point
        self.maj = (float(c @ st), float(st @ st))
        if algo == "fista":
            ln = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * sc.l_acc ** 2))
            sc.l_new, sc.beta = ln, (sc.l_acc - 1.0) / ln
        elif algo == "cp":
            sc.phi = 1.0 / np.sqrt(1.0 + 2.0 * cfg.cp_gamma * sc.tau)
            sc.sigma_new = sc.sigma / sc.phi
        cm = self._c()
        cm[0] = float(np.max(np.abs(c), initial=0.0))
        cm[1] = 0.0 if np.all(np.isfinite(cand)) else 1.0
        cm[2] = 0.0

    def _ph11(self):  # K1R
        sc = self.sc
        if sc.stop or sc.mode == 2:
            return
        self._radius(self._c()[0], self._c()[1] > 0)

    def _radius(self, m, nonfinite):
        sc = self.sc
        sc.nonfinite = nonfinite
        bound = np.inf if m == 0.0 else 1.0 / m
        sq, ty = sc.theta_sq, sc.theta_y
        mu = float(np.clip(ty / (self.lam * sq), -bound, bound)) if sq != 0.0 else 0.0
        d = self.y / self.lam - (mu * self.theta if sq != 0.0 else 0.0)
        sc.rsafe_sq = float(d @ d)
        if self.cfg.test == "safe":
            sc.radius = np.sqrt(sc.rsafe_sq)
        else:
            arg = sc.rsafe_sq - sc.shift_sq
            if arg < -1e-8:
                sc.status, sc.stop = -3, 6
            sc.radius = np.sqrt(max(arg, 0.0))

    def _ph12(self):  # K2
        sc, cfg = self.sc, self.cfg
        if sc.stop or sc.mode == 2:
            return
        A = self.active
        masked = np.zeros(A.size, dtype=bool)
        if cfg.strategy == "dynamic":
            masked = (1.0 - np.abs(self.cc[A])) - sc.radius > 1e-12
        self.mask = masked
        keep = A[~masked]
        cand = self.xn
        self.un = np.zeros(self.k)
        self.s_vec = np.zeros(self.k)
        if cfg.algorithm == "fista":
            self.un[keep] = cand[keep] + sc.beta * (cand[keep] - self.x[keep])
        elif cfg.algorithm == "cp":
            self.un[keep] = cand[keep] + sc.phi * (cand[keep] - self.x[keep])
        elif cfg.algorithm == "sparsa":
            self.s_vec[keep] = cand[keep] - self.x[keep]
        self.new_active = keep
        self.pen = float(np.sum(np.abs(cand[keep])))
        self.nnz = int(np.count_nonzero(cand[keep]))
        self.kept = int(keep.size)
        self.ss = float(self.s_vec[keep] @ self.s_vec[keep])
        self.dropped = bool(np.any(cand[A[masked]] != 0.0))

    def _ph13(self):  # K3A (+ the local sums K3S packs)
        sc, cfg = self.sc, self.cfg
        if sc.stop:
            return
        fix = sc.mode == 2
        if self.one:      # support built by K2S (all active units; the reduced list in a FIXUP trip)
            U = self.sup_units
            a = np.zeros(self.k)
            a[U] = self.xn[U]
            b = self.un if cfg.algorithm in ("fista", "cp") else self.s_vec
            self.Sa = self.D @ a
            self.Sb = self.D @ b
            return
        keep = self.new_active
        a = np.zeros(self.k)
        b = np.zeros(self.k)
        a[keep] = self.xn[keep]
        if cfg.algorithm in ("ista", "fista") and not fix:
            gone = np.setdiff1d(self.active, keep)
            a[gone] = self.xn[gone]
        if not fix:
            b = self.un if cfg.algorithm in ("fista", "cp") else self.s_vec
        self.Sa = self.D @ a
        self.Sb = self.D @ b

    def _ph14(self):  # K3S
        if self.sc.stop:
            return
        cm = self._c()
        cm[nat.CM_VEC:nat.CM_VEC + self.n] = self.Sa
        cm[nat.CM_VEC + self.n:nat.CM_VEC + 2 * self.n] = self.Sb
        if self.one:
            cm[nat.CM_SUM:nat.CM_SUM + 8] = [self.pen, self.nnz, 0.0, self.ss, 0.0, self.maj[0], self.maj[1], 0.0]
            base = nat.CM_VEC + 2 * self.n
            cm[base:base + nat.OC_SLOT * nat.OC_MAX_WORLD] = 0.0
            if self.sc.mode != 2:
                o = base + nat.OC_SLOT * self.rank
                cm[o:o + 6] = [cm[0], cm[1], cm[2], self.tmax, self.vmin, self.units]
            return
        cm[nat.CM_SUM:nat.CM_SUM + 8] = [self.pen, self.nnz, self.kept, self.ss, float(self.dropped),
                                         self.maj[0], self.maj[1], 0.0]

    def _ph15(self):  # K3B
        sc, cfg = self.sc, self.cfg
        if sc.stop:
            return
        cm = self._c()
        Sa = cm[nat.CM_VEC:nat.CM_VEC + self.n]
        Sb = cm[nat.CM_VEC + self.n:nat.CM_VEC + 2 * self.n]
        pen, nnz, kept, ss, dropped, mcs, mss = cm[nat.CM_SUM:nat.CM_SUM + 7]
        if self.one:
            kept, dropped = self.kept_local, float(self.dropped_oc)
        fix = sc.mode == 2 and not self.one
        qa = Sa - self.y
        algo = cfg.algorithm
        if algo == "fista":
            tn = None if fix else Sb - self.y
        elif algo == "cp":
            tn = None if fix else (self.theta + sc.sigma_new * (Sb - self.y)) / (1.0 + sc.sigma_new)
        else:
            tn = qa
        if sc.mode != 2:
            if sc.nonfinite:
                sc.status, sc.stop = -2, 6
                return
            if algo in ("ista", "fista"):
                f0 = 0.5 * sc.theta_sq
                bound = f0 + mcs + 0.5 * sc.L * mss
                if not (0.5 * float(qa @ qa) <= bound + 1e-12 * max(1.0, f0)):
                    sc.L *= cfg.backtrack_factor
                    sc.mode = 1
                    return
                if dropped > 0 and not self.one:
                    self.pending = tn
                    sc.mode = 2
                    return
            if self.one and dropped > 0:
                sc.mode = 2       # one collective: recompute both residuals on the reduced iterate
                return
        elif algo == "fista" and not self.one:
            tn = self.pending
        F = 0.5 * float(qa @ qa) + self.lam * pen
        gap = F - 0.5 * sc.yy + 0.5 * self.lam ** 2 * sc.rsafe_sq
        if algo == "fista":
            sc.l_acc = sc.l_new
        if algo == "cp":
            sc.tau, sc.sigma = sc.phi * sc.tau, sc.sigma_new
        if algo == "sparsa" and ss > 0.0:
            sc.L = float(np.clip(float(Sb @ Sb) / ss, cfg.bb_L_min, cfg.bb_L_max))
        sc.t += 1
        self.trace.append((sc.t, int(round(kept)), int(round(nnz)), F, gap))
        sc.moved = sc.moved or nnz > 0
        stop = 0
        if sc.moved and sc.have_fprev and abs(sc.f_prev - F) / max(F, 1e-300) < cfg.rel_tol:
            stop = 1
        elif cfg.gap_tol is not None and gap <= cfg.gap_tol:
            stop = 2
        elif (self.empty if self.one else round(kept) == 0):
            stop = 4
        elif sc.t >= cfg.max_iters:
            stop = 3
        sc.f_prev, sc.have_fprev = F, True
        self.theta = tn
        sc.theta_sq, sc.theta_y = float(tn @ tn), float(tn @ self.y)
        self.xp, self.x = self.x, self.xn
        if algo in ("fista", "cp"):
            self.u = self.un
        self.active = self.new_active
        sc.mode, sc.stop = 0, stop
        sc.gap = gap

    def _ph16(self):  # K2S: vectors and support over every active unit (reduced list in FIXUP)
        sc, cfg = self.sc, self.cfg
        if sc.stop:
            return
        fix = sc.mode == 2
        U = self.new_active if fix else self.active
        cand = self.xn
        self.un = np.zeros(self.k)
        self.s_vec = np.zeros(self.k)
        if cfg.algorithm == "fista":
            self.un[U] = cand[U] + sc.beta * (cand[U] - self.x[U])
        elif cfg.algorithm == "cp":
            self.un[U] = cand[U] + sc.phi * (cand[U] - self.x[U])
        elif cfg.algorithm == "sparsa":
            self.s_vec[U] = cand[U] - self.x[U]
        self.sup_units = U
        self.pen = float(np.sum(np.abs(cand[U])))
        self.nnz = int(np.count_nonzero(cand[U]))
        self.ss = float(self.s_vec[U] @ self.s_vec[U])
        if not fix:
            self.tmax, self.vmin, self.units = -np.inf, np.inf, float(U.size)
            if cfg.strategy == "dynamic" and U.size:
                v = 1.0 - np.abs(self.cc[U])
                b = self.un if cfg.algorithm in ("fista", "cp") else self.s_vec
                carries = (cand[U] != 0.0) | (b[U] != 0.0)
                self.vmin = float(np.min(v))
                if np.any(carries):
                    self.tmax = float(np.max(v[carries]))

    def _ph17(self):  # K1R1: gathered rank slots -> radius, dropped-nonzero, all-screened
        sc = self.sc
        if sc.stop or sc.mode == 2:
            return
        base = nat.CM_VEC + 2 * self.n
        sl = self._c()[base:base + nat.OC_SLOT * self.world].reshape(self.world, nat.OC_SLOT)
        self._radius(float(np.max(sl[:, 0])), float(np.max(sl[:, 1])) > 0)
        dyn = self.cfg.strategy == "dynamic"
        r = sc.radius
        self.dropped_oc = dyn and (float(np.max(sl[:, 3])) - r > 1e-12)
        self.empty = float(np.sum(sl[:, 5])) == 0.0 or (dyn and float(np.min(sl[:, 4])) - r > 1e-12)

    def _ph18(self):  # K2C: test and compaction
        sc, cfg = self.sc, self.cfg
        if sc.stop or sc.mode == 2:
            return
        A = self.active
        masked = np.zeros(A.size, dtype=bool)
        if cfg.strategy == "dynamic":
            masked = (1.0 - np.abs(self.cc[A])) - sc.radius > 1e-12
        self.mask = masked
        self.new_active = A[~masked]
        self.kept_local = int(self.new_active.size)

    @property
    def trace(self):
        if not hasattr(self, "_trace"):
            self._trace = []
        return self._trace
