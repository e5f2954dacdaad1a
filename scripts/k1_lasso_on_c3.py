"""c3's dictionary and observation solved as a plain Lasso (same bytes streamed by K1): isolates the
group path's cost.  python scripts/k1_lasso_on_c3.py"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from paper_1412_4080_b200.solver import Engine  # noqa: E402

w = wl.config3()
dic = ds.Dictionary(w.D, check_unit_norms=False)
L = ds.operator_norm(dic, tol=1e-11) ** 2 * (1 + 1e-6)
lam = 0.3 * float(abs(dic.correlate(w.y)).max())
cfg = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="dst3", max_iters=200, rel_tol=1e-300, L0=L)
eng = Engine(ds.Problem(dic, w.y, lam), cfg)
eng.setup()
ms = (C.c_float * 4)()
eng.L.dscr_solver_profile(eng.h, 40, eng.sptr, ms)
print("c3 data as Lasso, per-trip ms (K1, K2, K3a, K3b):", [round(v, 4) for v in ms])
