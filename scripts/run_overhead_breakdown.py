"""Where the host time of run() goes on c1 (warm): engine build (workspace, handle with both
graphs), setup, loop, readback.  python scripts/run_overhead_breakdown.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from paper_1412_4080_b200.solver import Engine  # noqa: E402

w = wl.config1()
dic = ds.Dictionary(w.D)
L = ds.operator_norm(dic, tol=1e-11) ** 2 * (1 + 1e-6)
cfg = ds.SolverConfig(algorithm=w.algorithm, strategy="dynamic", test=w.test, max_iters=w.max_iters,
                      rel_tol=1e-300, L0=L, gap_tol=w.gap_tol)
prob = ds.Problem(dic, w.y, w.lam)
ds.run(prob, cfg)
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e = Engine(prob, cfg)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    e.setup(); e.launch(0); sc = e.scalars()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    rows = e.trace_rows(sc.t)
    t3 = time.perf_counter()
    e.close()
    t4 = time.perf_counter()
    print(f"engine {1e3*(t1-t0):.2f} ms | setup+loop {1e3*(t2-t1):.2f} | readback {1e3*(t3-t2):.2f} | close {1e3*(t4-t3):.2f}")
