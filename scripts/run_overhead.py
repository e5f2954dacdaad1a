"""Wall time of the user-facing run() call (host API, warm) vs its device time: c1, c2, c3.
python scripts/run_overhead.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402

for name, w in (("c1", wl.config1()), ("c2", wl.config2(ratio=0.1)), ("c3", wl.config3())):
    dic = ds.Dictionary(w.D)
    part = ds.GroupPartition.build(dic, w.groups) if w.groups else None
    L = ds.operator_norm(dic, tol=1e-11) ** 2 * (1 + 1e-6)
    cfg = ds.SolverConfig(algorithm=w.algorithm, strategy="dynamic", test=w.test, max_iters=w.max_iters,
                          rel_tol=1e-300, L0=L, gap_tol=w.gap_tol)
    prob = ds.Problem(dic, w.y, w.lam, part)
    ds.run(prob, cfg)
    walls, devs = [], []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ds.run(prob, cfg)
        walls.append(time.perf_counter() - t0)
        devs.append(r.device_seconds)
    print(f"{name}: {r.iterations} it, run() wall {1e3 * np.median(walls):.2f} ms, device {1e3 * np.median(devs):.2f} ms")
