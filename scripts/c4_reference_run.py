"""One-off run of the REFERENCE itself (screenlab.run) on config 4 -> committed golden trace.

Build container only (the reference is not on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python scripts/c4_reference_run.py \
        [--n 8192 --k 262144 --seed 0 --ratio 0.2 --gap-tol 1e-5] --out tests/golden/c4_reference.npz

What it does (SURVEY §8(c) "reduced-precision configs"):
* generates c4 exactly as ``paper_1412_4080_b200.workloads.config4`` does (fp32 dictionary,
  fp64 unit-norm y, lam = ratio * max|D^T y| on the fp64 upcast);
* L = lambda_max(D D^T) * (1 + 1e-9) from an fp64 Gram (chunked) + eigvalsh, committed so
  the GPU side consumes the same float;
* runs the reference ``screenlab.run`` (``solvers.py:358-511``) on the fp64 upcast dictionary
  (``Dictionary(..., check_unit_norms=False)``), FISTA, dynamic DST3, rel_tol=1e-300, L0=L,
  with a hook that records r_SAFE^2 at theta_t with the pre-screening correlations (the
  BASELINE gap, SURVEY §8 a21 -- same as tests/golden/make_golden.py) and the support of
  (x_t, u_t);
* observes the reference's own trace (``SolveTrace.append``) and stops the run at the first t
  with gap_t <= gap_tol, which is the reference run with max_iters = t_hit;
* writes the per-iteration traces, the screened sets, x_t_hit (sparse) and the inputs' scalars.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import screenlab as sl  # noqa: E402  (reference, from PYTHONPATH)
from screenlab import solvers as sl_solvers  # noqa: E402

from paper_1412_4080_b200 import workloads as wl  # noqa: E402


class _Hit(Exception):
    pass


def gram_top_eig(D64, chunk=8192):
    n = D64.shape[0]
    G = np.zeros((n, n))
    for c0 in range(0, D64.shape[1], chunk):
        blk = D64[:, c0:c0 + chunk]
        G += blk @ blk.T
    return float(np.linalg.eigvalsh(G)[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--k", type=int, default=262144)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ratio", type=float, default=0.2)
    ap.add_argument("--gap-tol", type=float, default=1e-5)
    ap.add_argument("--max-iters", type=int, default=10000)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    t0 = time.time()
    w = wl.config4(seed=args.seed, ratio=args.ratio, n=args.n, k=args.k, gap_tol=args.gap_tol)
    n, k = w.D.shape
    D32 = w.D
    print(f"[{time.time()-t0:.0f}s] generated c4 {n}x{k} lam={w.lam!r}", flush=True)
    dic = sl.Dictionary(D32, check_unit_norms=False)          # fp64 upcast, F order (the reference's copy)
    del D32, w.D
    lmax_eig = gram_top_eig(dic.data)
    L = lmax_eig * (1.0 + 1e-9)
    print(f"[{time.time()-t0:.0f}s] ||D||^2 = {lmax_eig!r}, L = {L!r}", flush=True)
    prob = sl.Problem(dic, w.y, w.lam)
    cfg = sl.SolverConfig(algorithm="fista", strategy="dynamic", test="dst3", max_iters=args.max_iters,
                          rel_tol=1e-300, L0=L)
    lm = sl.lambda_max(prob)
    rec = {"rsafe_sq": [], "support": [], "corr_inf": [], "mu": []}
    masks = []
    last = {"x": None, "kept": None, "mask": None, "l": 1.0, "x_prev_full": None}
    yy = float(w.y @ w.y)

    def hook(info):
        ci = float(np.max(np.abs(info.corr), initial=0.0))
        mu, v = sl.dual_scale_lasso(prob, info.theta, corr_inf=ci)
        diff = prob.y / prob.lam - v
        rec["rsafe_sq"].append(float(diff @ diff))
        rec["corr_inf"].append(ci)
        rec["mu"].append(float(mu))
        # u_t exactly as update_fista forms it (solvers.py:220-224): u = x' + ((l-1)/l')(x' - x_old)
        x_full = np.zeros(k)
        x_full[info.kept] = info.x
        l_new = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * last["l"] ** 2))
        xo = last["x_prev_full"] if last["x_prev_full"] is not None else np.zeros(k)
        u_full = x_full + ((last["l"] - 1.0) / l_new) * (x_full - xo)
        last["l"] = float(l_new)
        kept_mask = np.zeros(k, bool)
        kept_mask[info.kept] = True
        rec["support"].append(int(np.count_nonzero(((x_full != 0) | (u_full != 0)) & kept_mask)))
        if info.mask is not None and info.mask.any():
            masks.append((info.t, info.kept[info.mask].copy()))
            x_full[info.kept[info.mask]] = 0.0
        last["x_prev_full"] = x_full
        last["x"], last["kept"], last["mask"] = info.x.copy(), info.kept.copy(), \
            (None if info.mask is None else info.mask.copy())

    trace_rows = []
    orig_append = sl_solvers.SolveTrace.append

    def append(self, t, kept, nnz, objective, flops, seconds):
        orig_append(self, t, kept, nnz, objective, flops, seconds)
        gap = objective - 0.5 * yy + 0.5 * prob.lam ** 2 * rec["rsafe_sq"][-1]
        trace_rows.append((t, kept, nnz, objective, gap))
        if t % 50 == 0:
            print(f"[{time.time()-t0:.0f}s] t={t} kept={kept} nnz={nnz} F={objective:.15e} gap={gap:.3e}",
                  flush=True)
        if gap <= args.gap_tol:
            raise _Hit()

    sl_solvers.SolveTrace.append = append
    t_run = time.time()
    hit = False
    try:
        sl.run(prob, cfg, iteration_hook=hook)
    except _Hit:
        hit = True
    finally:
        sl_solvers.SolveTrace.append = orig_append
    run_s = time.time() - t_run
    rows = np.array(trace_rows, dtype=np.float64)
    t_hit = int(rows[-1, 0])
    xk, kept, mask = last["x"], last["kept"], last["mask"]
    if mask is not None and mask.any():
        xk, kept = xk[~mask], kept[~mask]
    x_star = np.zeros(k)
    x_star[kept] = xk
    nz = np.flatnonzero(x_star)
    elim_mask = np.ones(k, bool)
    elim_mask[kept] = False
    eliminated = np.flatnonzero(elim_mask).astype(np.int64)
    ev_t = np.array([t for t, _ in masks], dtype=np.int64)
    ev_atoms = np.concatenate([a for _, a in masks]).astype(np.int64) if masks else np.empty(0, np.int64)
    ev_len = np.array([a.size for _, a in masks], dtype=np.int64)
    np.savez_compressed(
        args.out, n=n, k=k, seed=args.seed, ratio=args.ratio, gap_tol=args.gap_tol, lam=w.lam, L=L,
        lmax=lm.value, lmax_index=lm.atom_index, t_hit=t_hit, hit=hit,
        t=rows[:, 0].astype(np.int64), kept=rows[:, 1].astype(np.int64), nnz=rows[:, 2].astype(np.int64),
        objective=rows[:, 3], gap=rows[:, 4], rsafe_sq=np.array(rec["rsafe_sq"]),
        corr_inf=np.array(rec["corr_inf"]), mu=np.array(rec["mu"]), support=np.array(rec["support"]),
        x_idx=nz.astype(np.int64), x_val=x_star[nz], eliminated=eliminated,
        screen_event_t=ev_t, screen_event_len=ev_len, screen_event_atoms=ev_atoms)
    summary = {"config": {"n": n, "k": k, "seed": args.seed, "ratio": args.ratio, "gap_tol": args.gap_tol,
                          "algorithm": "fista", "test": "dst3"},
               "lam": w.lam, "L": L, "lambda_max": lm.value, "t_hit": t_hit, "hit": hit,
               "final_objective": float(rows[-1, 3]), "final_gap": float(rows[-1, 4]),
               "nnz": int(nz.size), "eliminated": int(eliminated.size), "reference_run_seconds": run_s,
               "iters_per_s_cpu": t_hit / run_s, "cpu": os.cpu_count(),
               "command": "PYTHONPATH=/root/reference/pkg/src python scripts/c4_reference_run.py " +
                          " ".join(sys.argv[1:])}
    print(json.dumps(summary), flush=True)
    with open(os.path.splitext(args.out)[0] + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
