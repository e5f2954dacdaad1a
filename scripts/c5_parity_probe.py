"""Probe: c5 batched solve vs the bf16-operand oracle and the fp64 oracle (stats only)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1412_4080_b200 as ds
from paper_1412_4080_b200 import workloads as wl
from paper_1412_4080_b200.batched import solve_batched
from oracle import batched_oracle as bo
from oracle import screen_oracle as so


def probe(w, dic, L, splits, picks, iters=100):
    D64 = dic.as_float64()
    t0 = time.time()
    res = solve_batched(dic, w.y, w.lam, L, iterations=iters, test="dst3", splits=splits, masks=True)
    print(f"solve {time.time() - t0:.1f}s kept min {res.kept.min()} mean {res.kept.mean():.0f}", flush=True)
    for j in picks:
        y, lam = w.y[:, j], float(w.lam[j])
        emu = bo.solve_bf16(D64, y, lam, L, iters, splits=splits)
        ref = so.solve(so.make_problem(D64, y, lam), so.Config(algorithm="fista", strategy="dynamic", test="dst3",
                       max_iters=iters, rel_tol=1e-300, L0=L, norm_aware=True))
        x = res.x_dense(j, D64.shape[1])
        el = res.eliminated(j)
        print(f"j={j:5d} kept gpu/emu/ref {res.kept[j]:6d} {emu.kept:6d} {D64.shape[1] - ref.eliminated.size:6d} "
              f"F-emu {abs(res.objective[j] - emu.objective) / emu.objective:.2e} "
              f"x-emu {np.linalg.norm(x - emu.x) / max(np.linalg.norm(emu.x), 1e-300):.2e} "
              f"F-ref {abs(res.objective[j] - ref.final_objective) / ref.final_objective:.2e} "
              f"emu-ref {abs(emu.objective - ref.final_objective) / ref.final_objective:.2e} "
              f"gpu\\emu {np.setdiff1d(el, emu.eliminated).size} emu\\gpu {np.setdiff1d(emu.eliminated, el).size} "
              f"gpu\\ref {np.setdiff1d(el, ref.eliminated).size}", flush=True)


if __name__ == "__main__":
    w, = [wl.config5(seed=0, n=128, k=1024, batch=256, nnz=8, ratio=0.4)]
    dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="bf16")
    L = float(np.linalg.norm(dic.as_float64(), 2) ** 2 * (1 + 1e-6))
    for s in (1, 2):
        print(f"== small 128x1024x256 ratio 0.4 splits {s}")
        probe(w, dic, L, s, range(0, 256, 17))
    w = wl.config5(seed=0)
    dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="bf16")
    nrm = ds.operator_norm(dic, tol=1e-11, max_iters=20000)
    L = nrm * nrm * (1.0 + 1e-6)
    print("== c5 bench batch splits 1")
    res = solve_batched(dic, w.y, w.lam, L, iterations=100, test="dst3", splits=1)
    picks = sorted(set(list(np.argsort(res.kept, kind="stable")[:12]) + list(range(0, 4096, 341))))
    probe(w, dic, L, 1, picks)
