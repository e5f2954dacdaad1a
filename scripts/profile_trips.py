"""Direct-launch iterations (dscr_solver_profile) of a workload, for ncu (graph kernels with
conditional nodes cannot be profiled per node): python scripts/profile_trips.py c3 [trips]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from timing_breakdown import workload  # noqa: E402
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200.solver import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
trips = int(sys.argv[2]) if len(sys.argv) > 2 else 40
w = workload(name)
dic = ds.Dictionary(w.D, check_unit_norms=False, dtype=w.dtype)
part = ds.GroupPartition.build(dic, w.groups) if w.groups else None
L = ds.operator_norm(dic, tol=1e-11) ** 2 * (1 + 1e-6)
cfg = ds.SolverConfig(algorithm=w.algorithm, strategy="dynamic", test=w.test, max_iters=w.max_iters,
                      rel_tol=1e-300, L0=L, gap_tol=w.gap_tol)
eng = Engine(ds.Problem(dic, w.y, w.lam, part), cfg)
eng.setup()
ms = (C.c_float * 4)()
eng.L.dscr_solver_profile(eng.h, trips, eng.sptr, ms)
print(name, "per-trip ms (K1, K2, K3a, K3b):", [round(v, 4) for v in ms])
